"""Step time of a bench.py suite workload (cfg1 / cfg2 / cfg4_*) at a given
batch under env-var tuning knobs.  SWEEP_ENV is a ';'-separated list of
settings, each a ','-separated list of NAME=VALUE (empty = defaults)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench

dev = torch.device("cuda", 0)
wname = os.environ.get("SWEEP_WL", "cfg1")
wl = dict(bench.WORKLOADS[wname])
for B in [int(x) for x in os.environ.get("SWEEP_B", str(wl["B"])).split(",")]:
    w = bench.make_workload(wl, B, 0, dev)
    for setting in os.environ.get("SWEEP_ENV", "").split(";"):
        kv = [s.split("=") for s in setting.split(",") if s]
        old = {k: os.environ.get(k) for k, _ in kv}
        for k, v in kv:
            os.environ[k] = v
        w.step()
        torch.cuda.synchronize()
        g, _ = bench.capture(w.step)
        run = g.replay if g is not None else w.step
        for _ in range(3):
            run()
        ms = bench.time_steps(run, 10)
        per = {}
        if os.environ.get("SWEEP_PEROP"):
            hbm, _ = bench.load_hbm_peak()
            dom, _ = w.attribution(5, hbm, {"dfma_tflops": 33.5, "dmma_tflops": 36.9, "source": "x"})
            per = {k: v["ms"] for k, v in dom["per_op"].items()}
        print(json.dumps({"wl": wname, "B": B, "env": setting, "ms": round(ms, 4), "per_op": per}), flush=True)
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        del g
    del w
    torch.cuda.empty_cache()
