#!/bin/bash
# one full ncu capture (source-level): profile_one.sh NAME WORKLOAD KERNEL_REGEX
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
PROF_WL=$2 timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$3" -c 1 \
  -o /tmp/$1 python scripts/profile_suite.py > gpurun_out/$1.log 2>&1
ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
ncu -i /tmp/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/$1_sass.csv 2>/dev/null
ncu -i /tmp/$1.ncu-rep --page details --print-details all > gpurun_out/$1_details.txt 2>/dev/null
ls -la gpurun_out | tail -5
