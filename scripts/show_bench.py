"""One-paragraph summary of bench.py JSON lines: python scripts/show_bench.py FILE..."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "no json", e)
        continue
    if d.get("impl") == "reference":
        print(f"{f}: REF value {d['value']:.4g} ms/step {d['ms_per_step']} sample: {d['cpu_baseline']['sample'][:90]} cores {d['cpu_baseline']['cores']}")
        continue
    r = d["roofline"]
    print(f"{f}: {d['config']['workload']} ms {d['ms_per_step']} value {d['value']:.4g} dom {r['kernel']} {r['kernel_ms']} "
          f"{r['bound']} frac {r['frac']} suite {d['suite_roofline']} clocks {d['clocks']['sm_mhz']} {d['clocks']['reasons']}")
    print(f"   launches {d['gpu_launches']} e2e {d['e2e']['value']:.4g} ({d['e2e']['ms_per_step']} ms) cpu {d['cpu_baseline']['value']:.4g} x{d['cpu_baseline']['cores']} peaks {d['fp64_peaks']['dfma_tflops']}/{d['fp64_peaks']['dmma_tflops']}")
    p = d.get("parity") or {}
    print(f"   parity {p.get('pass')} " + str({k: (v['max_rel_pinned_1e-12'], v['max_rel_floor_1e-6']) for k, v in p.get('outputs', {}).items()}))
    if d.get("scaling_proxy"):
        print("   proxy " + str({g: (v['ms_per_step'], v['efficiency']) for g, v in d['scaling_proxy'].items()}))
    if "per_op" in r:
        print("   per-op " + str({k: (v['ms'], v['frac']) for k, v in r['per_op'].items()}))
