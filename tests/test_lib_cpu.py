"""CPU tests of the product library boundary (no GPU needed).

The C ABI library must load, export every symbol include/*.h declares, and
reject invalid arguments with the reference's error class and wording before
touching the device.
"""
import ctypes as C
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def native():
    from paper_1204_5072_b200 import build

    build.build()
    from paper_1204_5072_b200 import _native

    return _native


def test_library_exports_every_declared_symbol(native):
    names = native.declared_symbols()
    assert len(names) >= 20
    lib = native.lib()
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", native.LIB_PATH], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert set(names) <= exported
    # nothing but the C ABI is exported
    assert all(s.startswith("lfg_") for s in exported if not s.startswith("_")), sorted(exported)[:10]


def test_abi_version_and_device_count(native):
    assert native.lib().lfg_abi_version() == 1
    assert native.device_count() >= 0


def test_sm100a_code_present(native):
    out = subprocess.run(["cuobjdump", "--list-elf", native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("L", [0, 2, 6, 100, 1000])
def test_kpz_rejects_bad_size(native, L):
    import paper_1204_5072_b200 as lfg

    with pytest.raises(lfg.InvalidArgument, match="power of two"):
        lfg.KpzLattice(L)


def test_kpz_rejects_small_for_dtr(native):
    import paper_1204_5072_b200 as lfg

    with pytest.raises(lfg.InvalidArgument, match="DtrPlan"):
        lfg.KpzLattice(32)


@pytest.mark.parametrize("p,q,msg", [(1.5, 0.0, "lie in"), (-0.1, 0.0, "lie in"), (0.5, 1.01, "lie in"),
                                     (0.0, 0.0, "positive"), (float("nan"), 0.0, "lie in")])
def test_kpz_rejects_bad_params(native, p, q, msg):
    # KpzParams::validate (kpz.hpp:19-26)
    import paper_1204_5072_b200 as lfg

    with pytest.raises(lfg.InvalidArgument, match=msg):
        lfg.KpzLattice(64, p, q)


def test_null_handle_rejected(native):
    lib = native.lib()
    assert lib.lfg_kpz_init_flat(None) == native.LFG_EINVAL
    assert b"null" in lib.lfg_last_error()


def test_header_compiles_as_c():
    src = "#include \"lfg.h\"\nint main(void){return lfg_abi_version()==1?0:1;}\n"
    tmp = "/tmp/lfg_hdr_test.c"
    with open(tmp, "w") as f:
        f.write(src)
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-c", "-I", os.path.join(ROOT, "include"), tmp,
                        "-o", "/tmp/lfg_hdr_test.o"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_sweep_origin_matches_oracle(native, oracle):
    # host-side DTr draws of the C ABI (used by the sharded driver) == oracle restatement
    from paper_1204_5072_b200.shard import StripPlan, sweep_origin

    for (L, bx, by) in ((2048, 1024, 128), (256, 64, 32), (1 << 16, 1024, 128)):
        pl = StripPlan(L, 1, bx, by)
        for s in range(20):
            ox, oy, sets = sweep_origin(pl, 12345, s)
            assert [ox, oy, *sets] == oracle.kpz_sweep_draw(L, bx, by, 12345, s).tolist()
