"""One-page summary of a full ncu capture reduced by scripts/profile_one.sh: key metrics from the raw
page and the per-region stall table of the SASS page.
python scripts/ncu_brief.py NAME "command / note" > profiles/NAME.txt  (reads gpurun_out/NAME_{raw,sass}.csv)"""
import csv
import subprocess
import sys

name, note = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
rows = list(csv.reader(open(f"gpurun_out/{name}_raw.csv")))
h, v = rows[0], rows[2] if len(rows) > 2 else rows[1]
col = {c: i for i, c in enumerate(h)}
keys = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__waves_per_multiprocessor",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
print(f"ncu --set full --import-source on --clock-control none (scripts/profile_one.sh {name}); {note}\n")
units = rows[1] if len(rows) > 2 else [""] * len(h)
for k in keys:
    if k in col:
        print(f"{k} {v[col[k]]} {units[col[k]]}")
print("\nstall samples per SASS region between barriers (scripts/sass_regions.py; regions >= 0.2% of samples):")
sys.stdout.flush()
subprocess.run([sys.executable, "scripts/sass_regions.py", f"gpurun_out/{name}_sass.csv"])
