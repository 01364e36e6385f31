"""One line per kernel launch of an ncu report: duration, DRAM traffic and
achieved GB/s, warps, issue, registers, grid -- the profiles/ summary format.
python scripts/ncu_summary.py REP [REP ...]"""
import csv
import io
import subprocess
import sys

M = {"t": "gpu__time_duration.sum", "rd": "dram__bytes_read.sum", "wr": "dram__bytes_write.sum",
     "dram": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
     "warps": "sm__warps_active.avg.pct_of_peak_sustained_active",
     "issue": "smsp__issue_active.avg.pct_of_peak_sustained_active",
     "regs": "launch__registers_per_thread", "grid": "launch__grid_size", "block": "launch__block_size",
     "smem": "launch__shared_mem_per_block_dynamic"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-3, "ms": 1.0, "ns": 1e-6}

for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    idx = {k: h.index(v) for k, v in M.items() if v in h}
    name = h.index("Kernel Name")
    print(f"# {rep}")
    for r in rows[2:]:
        def val(k):
            v = float(r[idx[k]].replace(",", ""))
            return v * SCALE.get(units[idx[k]].split("/")[0], 1.0)
        ms = val("t")
        traffic = val("rd") + val("wr")
        kn = r[name].replace("(anonymous namespace)::", "").replace("unnamed>::", "")
        kn = kn[:70]
        print(f"{kn:<70} {ms:8.3f} ms  DRAM rd {val('rd') / 1e9:6.3f} GB wr {val('wr') / 1e9:6.3f} GB "
              f"= {traffic / ms / 1e6:7.1f} GB/s ({val('dram'):5.1f}% peak)  warps {val('warps'):5.1f}%  "
              f"issue {val('issue'):5.1f}%  regs {int(val('regs'))}  grid {int(val('grid'))}x{int(val('block'))}  "
              f"smem {val('smem') / 1e3:.0f} KB")
        sys.stdout.flush()
