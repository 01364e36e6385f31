"""Accuracy probe for config-3 gradients: oracle (reference tape route, fp64)
and the CUDA fast path vs an extended-precision (x87 long double) evaluation
of the same mathematics, on one small instance.

    python scripts/precision_probe.py [n] [seg]

Prints, per quantity, the max elementwise error normalised by max|exact|
(absolute-relative) and the elementwise relative error with floors 1e-12 and
1e-6 of max|exact|, for both implementations.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import oracle as orc
from tests import common as cm

LD = np.longdouble


def dense_lower(Lb, n, k):
    D = np.zeros((n, n), dtype=LD)
    for r in range(k + 1):
        idx = np.arange(n - r)
        D[idx + r, idx] = Lb[: n - r, r].astype(LD)
    return D


def inv_ld(A):
    n = A.shape[0]
    M = np.concatenate([A.copy(), np.eye(n, dtype=LD)], axis=1)
    for c in range(n):
        M[c] /= M[c, c]
        f = M[:, c].copy()
        f[c] = 0
        M -= np.outer(f, M[c])
    return M[:, n:]


def exact(L, y, tau2, k):
    B, n, _ = L.shape
    out_l, out_lb, out_tb = [], [], []
    s = LD(1) / LD(tau2)
    for b in range(B):
        Ld = dense_lower(L[b], n, k)
        A = Ld @ Ld.T + s * np.eye(n, dtype=LD)
        Ai = inv_ld(A)
        yv = y[b].astype(LD)
        u = Ai @ yv
        G = -((Ai + s * s * np.outer(u, u)) @ Ld) + np.diag(LD(1) / np.diag(Ld))
        lb = np.zeros((n, k + 1), dtype=LD)
        for r in range(k + 1):
            idx = np.arange(n - r)
            lb[: n - r, r] = G[idx + r, idx]
        # loss via the same closed form as the reference objective
        sign, logdetA = np.linalg.slogdet(A.astype(np.float64))  # only for a rough loss check
        out_lb.append(lb)
        tb = (-LD(n) / (2 * LD(tau2)) + yv @ yv / (2 * LD(tau2) ** 2) + np.trace(Ai) / (2 * LD(tau2) ** 2)
              - (yv @ u) / LD(tau2) ** 3 + (u @ u) / (2 * LD(tau2) ** 4))
        out_tb.append(tb)
    return np.array(out_lb), np.array(out_tb)


def report(name, got, ex):
    got = np.asarray(got, dtype=LD)
    M = np.max(np.abs(ex))
    d = np.abs(got - ex)
    absrel = float(np.max(d) / M)
    out = [f"{name:10s} max|d|/M={absrel:.2e}"]
    for fl in (1e-12, 1e-6):
        den = np.maximum(np.maximum(np.abs(got), np.abs(ex)), fl * M)
        out.append(f"rel(floor {fl:g})={float(np.max(d / den)):.2e}")
    print("  ".join(out))


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 400
    seg = int(sys.argv[2]) if len(sys.argv) > 2 else 128
    B, k, tau2 = 3, 16, 0.01
    rng = np.random.default_rng(11)
    L = cm.config_factor(rng, B, n, k)
    y = rng.normal(0, 1, (B, n))
    lb_ex, tb_ex = exact(L, y, tau2, k)
    o = orc.Oracle("restatement")
    _, lb_o, tb_o, _, _ = o.marginal_likelihood_grad(L, y, tau2)
    print(f"n={n} k={k} B={B}")
    report("oracle", lb_o, lb_ex)
    report("oracle tb", tb_o, tb_ex)
    try:
        import torch
        if torch.cuda.is_available():
            from paper_1902_10078_b200 import api
            from tests.gpu_adapter import GpuOracle
            api.set_segment_rows(seg)
            _, lb_g, tb_g, _, _ = GpuOracle(tile=1).marginal_likelihood_grad(L, y, tau2)
            report("gpu fast", lb_g, lb_ex)
            report("gpu tb", tb_g, tb_ex)
            _, lb_g2, _, _, _ = GpuOracle(tile=32).marginal_likelihood_grad(L, y, tau2)
            report("gpu gener", lb_g2, lb_ex)
    except ImportError:
        pass




def sweep_burn():
    """BGM_DEBUG=2: max burn-in deviation and gpu error vs exact per segment size."""
    import torch
    from paper_1902_10078_b200 import api
    from tests.gpu_adapter import GpuOracle
    n, B, k, tau2 = 2048, 3, 16, 0.01
    rng = np.random.default_rng(12)
    L = cm.config_factor(rng, B, n, k)
    y = rng.normal(0, 1, (B, n))
    o = orc.Oracle("restatement")
    _, lb_o, _, _, _ = o.marginal_likelihood_grad(L, y, tau2)
    for seg in (0, 256, 512, 1024):
        api.set_segment_rows(seg)
        api.debug_repairs(reset=True)
        _, lb_g, _, _, _ = GpuOracle(tile=1).marginal_likelihood_grad(L, y, tau2)
        torch.cuda.synchronize()
        reps, dev = api.debug_repairs(with_dev=True)
        M = np.abs(lb_o).max()
        print(f"seg={seg} repairs={reps} max_dev={dev:.2e} gpu-vs-oracle max|d|/M={np.abs(lb_g - lb_o).max() / M:.2e} "
              f"rel={cm.max_rel_err(lb_g, lb_o):.2e}")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "burn":
        sweep_burn()
    else:
        main()
