#!/bin/bash
# full ncu captures (source-level) of the top config-4 kernels; the reports are
# reduced to their raw and SASS-source CSV pages on the box (size limit)
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
cap() {  # name workload kernel-regex
  PROF_WL=$2 timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$3" -c 1 \
    -o /tmp/$1 python scripts/profile_suite.py > gpurun_out/$1.log 2>&1
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/$1_sass.csv 2>/dev/null
}
cap r02_chol_mw128 cfg4_k128_f64 '^k_chol_mw$'
cap r02_vsub64 cfg4_k64_f64 '^k_vsub_dmma$'
cap r02_wsolve64 cfg4_k64_f64 '^k_solve$'
ls -la gpurun_out
