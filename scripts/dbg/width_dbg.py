import os, sys
sys.path.insert(0, os.getcwd())
import paper_1204_5072_b200 as lfg
for L, bx, by in [(256, 128, 64), (1024, 0, 0)]:
    try:
        with lfg.KpzLattice(L, 1.0, 0.0, 1, block_x=bx, block_y=by) as k:
            k.make_flat_slopes()
            print("flat ok", flush=True)
            print(L, "w2", k.interface_width(), flush=True)
            k.sweep(1)
            print(L, "w2 after", k.interface_width(), flush=True)
    except Exception as e:
        print("ERR", L, type(e).__name__, e, flush=True)
