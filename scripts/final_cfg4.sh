cd /root/repo 2>/dev/null || cd $GRAFT_REPO_ROOT
T=r2i
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${T}_gputests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_gputests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_smoke.log
for w in cfg4_k64_f64 cfg4_k64_f32 cfg4_k128_f64 cfg4_k128_f32; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/${T}_bench_$w.json 2> gpurun_out/${T}_bench_$w.err
done
bash scripts/profile_cfg4.sh
bash scripts/profile_many.sh "r02_vchol128 cfg4_k128_f64 ^k_vchol_dmma\$" "r02_subset128 cfg4_k128_f64 ^k_subset_mw\$"
