"""Per-operator suite timing for BASELINE.json configs 1-4.

Each operator is timed as its own API call on device-resident, tile-32 data
(CUDA events, median of `--reps` after one warm-up); the suite time is the
sum.  Roofline per op = max(bytes / HBM, flops / FP64) with the per-row
counts of SURVEY.md §8(d); HBM from MEASURED_PEAKS.json, FP64 37.2 TF
(fp32 74.4 TF) nominal.  Prints one JSON object per config.

    python scripts/bench_ops.py [--configs 1,2,3,4] [--reps 5]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1902_10078_b200 as bgm  # noqa: E402
from paper_1902_10078_b200 import api  # noqa: E402

FP64_TF = 37.2
FP32_TF = 74.4


def hbm_gbs():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6549.4


# per band-row (flops, bytes at fp64); SURVEY.md §8(d)
def counts(op, k, wa=None, wb=None, w=None):
    if op == "cholesky":
        return (k + 1) ** 2, 16 * (k + 1)
    if op == "solve_vec":
        return 2 * k + 1, 8 * (k + 3)
    if op == "log_det":
        return 1, 8
    if op == "subset":
        return 2 * k * (k + 1) + k + 2, 16 * (k + 1)
    if op == "product":
        return 2 * wa * wb, 8 * (2 * wa + 2 * wb - 1)
    if op == "llt_lower":
        return (k + 1) * (k + 2), 16 * (k + 1)
    if op == "band_vec":
        return 2 * w, 8 * (w + 2)
    if op == "vjp_cholesky":
        return 2 * k * (k + 1) + 4 * k + 2, 24 * (k + 1)
    if op == "vjp_solve_vec":
        return 3 * k + 2, 16 * (k + 1) + 24
    if op == "vjp_log_det":
        return 1, 8 + 8 * (k + 1)
    if op == "vjp_subset":
        return 4 * k * (k + 1) + 2 * (k + 1) + 3 * k + 7, 32 * (k + 1)
    if op == "vjp_product":
        return 4 * wa * wb, 8 * (3 * wa + 3 * wb - 1)
    if op == "vjp_band_vec":
        return 3 * w, 8 * (2 * w + 3)
    raise KeyError(op)


def timeit(fn, reps):
    """Median per-call time.  Ops shorter than 2 ms are timed as `inner`
    back-to-back API calls between two events (the host enqueues call i+1
    while call i runs, as a caller looping over batches would), so the
    figure is the op's device throughput rather than Python launch latency;
    a host-bound op still shows as host-bound."""
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    t_first = e0.elapsed_time(e1)
    if t_first > 2000:  # very slow op: one timed rep is enough
        return t_first
    inner = 1 if t_first > 2.0 else max(2, min(20, int(4.0 / max(t_first, 1e-3))))
    out = []
    for _ in range(reps):
        e0.record()
        for _ in range(inner):
            fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) / inner)
    return statistics.median(out)


def factor(B, n, k, dtype, dev, off_std, seed, tile=32):
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    L = bgm.Bands.empty(B, n, k, 0, tile=1, dtype=torch.float64, device=dev)
    L.data.normal_(0.0, off_std, generator=g)
    L.data[:, :, 0].uniform_(1.0, 2.0, generator=g)
    for r in range(1, k + 1):
        L.data[:, n - r:, r] = 0.0
    out = L.to_tile(tile) if tile == 32 else L
    if dtype == torch.float32:
        out = bgm.Bands(out.data.float(), B, n, k, 0, tile)
    return out


def normal_band(B, n, lo, up, dtype, dev, seed, tile=32):
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    X = bgm.Bands.empty(B, n, lo, up, tile=tile, dtype=dtype, device=dev)
    X.data.normal_(0.0, 1.0, generator=g)
    return X


def normal_vec(B, n, dtype, dev, seed, tile=32):
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    v = bgm.Vecs.empty(B, n, tile=tile, dtype=dtype, device=dev)
    v.data.normal_(0.0, 1.0, generator=g)
    return v


def report(name, B, n, dtype, ops, hbm):
    peak_flops = (FP32_TF if dtype == torch.float32 else FP64_TF) * 1e12
    scale = 0.5 if dtype == torch.float32 else 1.0
    rows = []
    tot_ms = tot_roof = 0.0
    for op, ms, fl, by in ops:
        roof = max(by * scale * B * n / (hbm * 1e9), fl * B * n / peak_flops) * 1e3
        rows.append({"op": op, "ms": round(ms, 4), "roofline_ms": round(roof, 4),
                     "frac": round(roof / ms, 4), "band_rows_per_s": round(B * n / (ms / 1e3), 1)})
        tot_ms += ms
        tot_roof += roof
    return {"config": name, "B": B, "n": n, "dtype": str(dtype).replace("torch.", ""),
            "suite_ms": round(tot_ms, 4), "suite_roofline_ms": round(tot_roof, 4),
            "suite_frac": round(tot_roof / tot_ms, 4), "band_rows_per_s": round(B * n / (tot_ms / 1e3), 1),
            "ops": rows}


def cfg1(dev, reps, hbm):
    B, n, k = 4096, 2048, 4
    L = factor(B, n, k, torch.float64, dev, 0.1, 11)
    Q = bgm.product_band_band_restricted(L, bgm.T(L), k, 0)
    b = normal_vec(B, n, torch.float64, dev, 12)
    Lq = bgm.cholesky(Q)
    x = bgm.solve_vec(Lq, b)
    ops = []
    for op, fn, c in (("cholesky", lambda: bgm.cholesky(Q, check=False), counts("cholesky", k)),
                      ("solve_vec L", lambda: bgm.solve_vec(Lq, b, False, check=False), counts("solve_vec", k)),
                      ("solve_vec Lt", lambda: bgm.solve_vec(Lq, x, True, check=False), counts("solve_vec", k)),
                      ("log_det", lambda: bgm.log_det_from_cholesky(Lq, check=False), counts("log_det", k))):
        ops.append((op, timeit(fn, reps), *c))
    return report("cfg1", B, n, torch.float64, ops, hbm)


def cfg2(dev, reps, hbm):
    B, n, k = 512, 65536, 8
    L = normal_band(B, n, k, 0, torch.float64, dev, 21)
    Lt = L.transpose()
    A = normal_band(B, n, 8, 8, torch.float64, dev, 22)
    Bm = normal_band(B, n, 3, 3, torch.float64, dev, 23)
    v = normal_vec(B, n, torch.float64, dev, 24)
    ops = []
    P1 = bgm.product_band_band(L, bgm.T(L))
    ops.append(("L.Lt full (8,8)", timeit(lambda: bgm.product_band_band(L, bgm.T(L)), reps),
                2 * (k + 1) ** 2, 8 * (3 * k + 2)))
    del P1
    P2 = bgm.product_band_band(A, Bm)
    ops.append(("A(8,8).B(3,3)", timeit(lambda: bgm.product_band_band(A, Bm), reps),
                *counts("product", k, wa=17, wb=7)))
    del P2
    ops.append(("A.v", timeit(lambda: bgm.product_band_vec(A, v), reps), *counts("band_vec", k, w=17)))
    Pb1 = normal_band(B, n, 8, 8, torch.float64, dev, 25)
    ops.append(("vjp L.Lt", timeit(lambda: bgm.vjp_product_band_band(L, Lt, Pb1), reps),
                *counts("vjp_product", k, wa=9, wb=9)))
    del Pb1
    Pb2 = normal_band(B, n, 11, 11, torch.float64, dev, 26)
    ops.append(("vjp A.B", timeit(lambda: bgm.vjp_product_band_band(A, Bm, Pb2), reps),
                *counts("vjp_product", k, wa=17, wb=7)))
    del Pb2
    pv = normal_vec(B, n, torch.float64, dev, 27)
    ops.append(("vjp A.v", timeit(lambda: bgm.vjp_product_band_vec(A, v, pv, False), reps),
                *counts("vjp_band_vec", k, w=17)))
    return report("cfg2", B, n, torch.float64, ops, hbm)


def wide(dev, reps, hbm, k, dtype, B=64, n=32768, tag="cfg4", with_vjp_recurrences=False):
    """Config 4 in the reference layout (tile 1): one CTA / warp per
    (matrix, segment) reads whole contiguous columns."""
    t = 1
    L0 = factor(B, n, k, dtype, dev, 0.02 / k ** 0.5, 41 + k, tile=t)
    Q = bgm.product_band_band_restricted(L0, bgm.T(L0), k, 0)
    L = bgm.cholesky(Q)
    b = normal_vec(B, n, dtype, dev, 42, tile=t)
    x1 = bgm.solve_vec(L, b)
    x2 = bgm.solve_vec(L, x1, True)
    S = bgm.sparse_inverse_subset(L)
    Lb = normal_band(B, n, k, 0, dtype, dev, 43, tile=t)
    Sb = normal_band(B, n, k, 0, dtype, dev, 44, tile=t)
    sb = normal_vec(B, n, dtype, dev, 45, tile=t)
    ops = []
    spec = [("cholesky", lambda: bgm.cholesky(Q, check=False), counts("cholesky", k)),
            ("solve_vec L", lambda: bgm.solve_vec(L, b, False, check=False), counts("solve_vec", k)),
            ("solve_vec Lt", lambda: bgm.solve_vec(L, x1, True, check=False), counts("solve_vec", k)),
            ("log_det", lambda: bgm.log_det_from_cholesky(L, check=False), counts("log_det", k)),
            ("subset", lambda: bgm.sparse_inverse_subset(L, check=False), counts("subset", k)),
            ("vjp_solve_vec L", lambda: bgm.vjp_solve_vec(L, x1, sb, False, check=False), counts("vjp_solve_vec", k)),
            ("vjp_solve_vec Lt", lambda: bgm.vjp_solve_vec(L, x2, sb, True, check=False), counts("vjp_solve_vec", k)),
            ("vjp_log_det", lambda: bgm.vjp_log_det_from_cholesky(L, 1.0), counts("vjp_log_det", k))]
    if with_vjp_recurrences:
        spec += [("vjp_cholesky", lambda: bgm.vjp_cholesky(L, Lb), counts("vjp_cholesky", k)),
                 ("vjp_subset", lambda: bgm.vjp_sparse_inverse_subset(L, S, Sb, check=False), counts("vjp_subset", k))]
    for op, fn, c in spec:
        ops.append((op, timeit(fn, reps), *c))
    return report(f"{tag} k={k}" + ("" if with_vjp_recurrences else " (without vjp_cholesky / vjp_subset)"),
                  B, n, dtype, ops, hbm)


def cfg3_ops(dev, reps, hbm):
    """The reference composition of config 3, op by op (the fused step is bench.py)."""
    B, n, k, tau2 = 256, 65536, 16, 0.01
    L = factor(B, n, k, torch.float64, dev, 0.1, 31)
    y = normal_vec(B, n, torch.float64, dev, 32)
    Q = bgm.product_band_band_restricted(L, bgm.T(L), k, 0)
    Lp = bgm.cholesky(Q)
    w = bgm.solve_vec(Lp, y)
    Lb = normal_band(B, n, k, 0, torch.float64, dev, 33)
    G = normal_band(B, n, k, 0, torch.float64, dev, 34)
    Lt = L.transpose()
    ops = []
    spec = (("L.Lt lower", lambda: bgm.product_band_band_restricted(L, bgm.T(L), k, 0), counts("llt_lower", k)),
            ("cholesky x2", lambda: (bgm.cholesky(Q, check=False), bgm.cholesky(Q, check=False)),
             tuple(2 * c for c in counts("cholesky", k))),
            ("solve_vec", lambda: bgm.solve_vec(Lp, y, False, check=False), counts("solve_vec", k)),
            ("log_det x2", lambda: (bgm.log_det_from_cholesky(Lp, check=False),) * 2,
             tuple(2 * c for c in counts("log_det", k))),
            ("vjp_solve_vec", lambda: bgm.vjp_solve_vec(Lp, w, y, False, check=False), counts("vjp_solve_vec", k)),
            ("vjp_log_det x2", lambda: (bgm.vjp_log_det_from_cholesky(Lp, 1.0), bgm.vjp_log_det_from_cholesky(Lp, 1.0)),
             tuple(2 * c for c in counts("vjp_log_det", k))),
            ("vjp_cholesky x2", lambda: (bgm.vjp_cholesky(Lp, Lb), bgm.vjp_cholesky(Lp, Lb)),
             tuple(2 * c for c in counts("vjp_cholesky", k))),
            ("vjp L.Lt (dL)", lambda: bgm.vjp_product_band_band(L, Lt, G), (612, 544)))
    for op, fn, c in spec:
        ops.append((op, timeit(fn, reps), *c))
    return report("cfg3 (reference composition, op by op)", B, n, torch.float64, ops, hbm)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,4")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--no-wide-vjp", dest="wide_vjp", action="store_false",
                    help="skip the wide vjp_cholesky / vjp_subset")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    hbm = hbm_gbs()
    todo = args.configs.split(",")
    for c in todo:
        t0 = time.time()
        if c == "1":
            res = cfg1(dev, args.reps, hbm)
        elif c == "2":
            res = cfg2(dev, args.reps, hbm)
        elif c == "3":
            res = cfg3_ops(dev, args.reps, hbm)
        elif c == "4":
            for k in (64, 128):
                for dt in (torch.float64, torch.float32):
                    res = wide(dev, args.reps, hbm, k, dt, with_vjp_recurrences=args.wide_vjp)
                    res["wall_s"] = round(time.time() - t0, 1)
                    print(json.dumps(res), flush=True)
                    t0 = time.time()
            continue
        else:
            continue
        res["wall_s"] = round(time.time() - t0, 1)
        print(json.dumps(res), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
