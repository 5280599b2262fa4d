#!/usr/bin/env bash
# Compile kpz_kernels.cu alone for sm_100a and report, for the production phase
# kernel (p = 1, 1024-wide, NT = 2, multi-warp, chained), registers and the
# number of uniform-datapath / vector instructions in its SASS -- the round loop
# loses the uniform datapath on some code shapes.
# Usage: bash scripts/kpz_sass_stats.sh [extra nvcc -D flags]
set -e
OUT=${TMPDIR:-/tmp}/kpz_sass; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -cubin -Xptxas -v "$@" \
    -o $OUT/k.cubin paper_1204_5072_b200/csrc/kpz_kernels.cu 2> $OUT/ptxas.log
SYM=$(cuobjdump -sass $OUT/k.cubin | grep -o "Function : _ZN3lfg20kpz_dtr_phase_kernelILb0ELb1ELi2ELb1ELb0ELb1EEEvNS_12KpzPhaseArgsE" | head -1 | cut -d' ' -f3)
cuobjdump -sass -fun "$SYM" $OUT/k.cubin > $OUT/k.sass
echo "regs: $(grep -A2 "$SYM" $OUT/ptxas.log | grep -o "Used [0-9]* registers")"
echo "insts: $(grep -cE '^\s+/\*[0-9a-f]{4}\*/' $OUT/k.sass)  uniform: $(grep -cE '/\*[0-9a-f]{4}\*/\s+(@!?U?P[0-9T] )?U[A-Z0-9]+' $OUT/k.sass)  BRA.U: $(grep -c 'BRA.U' $OUT/k.sass)  LDS: $(grep -c ' LDS' $OUT/k.sass)"
