#!/bin/bash
# ncu --set full capture of the config-2 / config-3 staged product kernels,
# the tile-32 band x vector kernels and the narrow k = 16 recurrences
# (Cholesky, solves, vjp_cholesky) at full size; summarised by
# scripts/ncu_summary.py into profiles/.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
TAG=${TAG:-r01}
PROF_B=${PROF_B:-256} timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:'k_stream|k_band_vec32|k_vjp_band_vec32' -o gpurun_out/${TAG}_products python scripts/profile_products.py \
  > gpurun_out/${TAG}_products_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:'k_chol<|k_cholI|k_chol$|k_solve<|k_solveI|k_vchol<|k_vcholI' -c 6 -o gpurun_out/${TAG}_narrow \
  python scripts/time_narrow.py 0 > gpurun_out/${TAG}_narrow_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_vchol' -c 1 \
  -o gpurun_out/${TAG}_vchol python scripts/time_narrow_vchol.py 16 > gpurun_out/${TAG}_vchol_ncu.log 2>&1
python scripts/ncu_summary.py gpurun_out/${TAG}_products.ncu-rep gpurun_out/${TAG}_narrow.ncu-rep \
  gpurun_out/${TAG}_vchol.ncu-rep > gpurun_out/${TAG}_ops_ncu.txt 2>&1
# full reports are large: keep the summary (and the product report, for source-level reading)
rm -f gpurun_out/${TAG}_narrow.ncu-rep gpurun_out/${TAG}_vchol.ncu-rep
ls -la gpurun_out | tail -5
