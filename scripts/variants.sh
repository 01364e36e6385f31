#!/bin/bash
# Build and time compile-time variants of the library side by side.
#   build:  scripts/variants.sh build NAME "-DFOO=1 ..."
#   run:    scripts/variants.sh run NAME [NAME...]     (on the GPU box)
cd "$(dirname "$0")/.." || exit 1
PKG=paper_1902_10078_b200
if [ "$1" = build ]; then
  make -s -C $PKG BUILD=$PWD/$PKG/build_var/$2 LIB=$PWD/$PKG/build_var/$2/libbandgm_b200.so XFLAGS="$3" -j8
  exit $?
fi
shift
mkdir -p gpurun_out
for v in "$@"; do
  lib=$PWD/$PKG/build_var/$v/libbandgm_b200.so
  [ "$v" = main ] && lib=$PWD/$PKG/libbandgm_b200.so
  echo "== $v"
  BGM_LIBRARY=$lib timeout 600 python bench.py --no-cpu --no-e2e --steps 5 ${BENCH_ARGS} > gpurun_out/var_$v.log 2>&1
  grep -o '"ms_per_step": [0-9.]*' gpurun_out/var_$v.log; grep -o '"kernel_ms": {[^}]*}' gpurun_out/var_$v.log
done
