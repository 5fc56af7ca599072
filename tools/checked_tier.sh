#!/bin/bash
# Checked-build tier (stands in for compute-sanitizer, which is closed on the
# GPU pool): build libkatzb200 with -DKZ_CHECKED=1 (device bounds checks that
# trap, bounded spin-waits, red zones between workspace slices) and run the
# kernel-family workload plus the GPU test suite against it with poisoned
# (0xFF) workspaces and red-zone verification after every call.
set -o pipefail
out=gpurun_out/checked
mkdir -p $out
LIBC=build/variants/checked/libkatzb200.so
if [ ! -f $LIBC ]; then
  make -C paper_1912_06525_b200/csrc -j8 EXTRA="-DKZ_CHECKED=1" OBJDIR=$PWD/build/checked OUT=$PWD/$LIBC > $out/build.log 2>&1
fi
KZ_LIB_PATH=$LIBC timeout 900 python tools/sanitize_workload.py > $out/workload.log 2>&1; echo "workload rc=$? $(grep -c '^ok' $out/workload.log) steps"
KZ_LIB_PATH=$LIBC KZ_K1_SLICE_MB=0.1 KZ_K1_MINDEG=16 KZ_SANITIZE_PART=cg timeout 900 python tools/sanitize_workload.py > $out/workload_colblock.log 2>&1; echo "workload_colblock rc=$?"
KZ_LIB_PATH=$LIBC KZ_GRAPHS=1 timeout 900 python tools/sanitize_workload.py > $out/workload_graphs.log 2>&1; echo "workload_graphs rc=$?"
KZ_LIB_PATH=$LIBC timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest_gpu rc=$?"; tail -3 $out/pytest_gpu.log
