"""Host-buffer entry points: the call a user with data in host memory makes.

The reference's API is host-resident (Eigen storage).  For batches, the
drop-in keeps that contract and hides the PCIe traffic behind compute: the
batch is cut into chunks of whole matrices that flow through three stages
on three streams -- H2D copy, fused sweeps, D2H copy -- over a small ring of
device buffers, so the two copy engines run back to back in both directions
(PCIe Gen5 is full duplex) and the kernels hide behind them.
"""
from __future__ import annotations

import torch

from .api import Bands, Vecs, marginal_likelihood_grad, new_status


def marginal_likelihood_grad_host(L_host: torch.Tensor, y_host: torch.Tensor, tau2: float,
                                  out_host=None, chunk: int = 16, streams: int = 4, device=None,
                                  tile: int = 32):
    """Config-3 learning step on host buffers.

    L_host: (B, n, k+1) float64, the reference storage block per matrix
    (ideally pinned); y_host: (B, n).  Returns host (loss[B], l_bar, tau2_bar[B]).
    With tile 32 each chunk is re-interleaved on the device (32 matrices side
    by side) for the one-thread-per-unit sweeps and L_bar is brought back to
    the reference layout before the copy out; tile 1 feeds the reference
    layout to the kernels directly.
    """
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    B, n, w = L_host.shape
    k = w - 1
    if out_host is None:
        pin = L_host.is_pinned()
        out_host = (torch.empty(B, dtype=torch.float64, pin_memory=pin),
                    torch.empty_like(L_host, pin_memory=pin),
                    torch.empty(B, dtype=torch.float64, pin_memory=pin))
    loss_h, lbar_h, tbar_h = out_host
    if tile not in (1, 32):
        raise ValueError("tile must be 1 or 32")
    chunk = max(1, min(chunk, B))
    depth = max(2, streams)
    # Three stages on three streams -- copy in, compute, copy out -- over a ring of `depth` buffer sets:
    # the H2D engine streams chunk after chunk without waiting for kernels or D2H, the D2H engine drains
    # finished chunks concurrently (PCIe is full duplex), and the kernels hide behind both.  (One stream
    # per chunk, the first version, left the order of the copies to the hardware queues: 57-72 ms per
    # config-3 step depending on the box against ~46 ms of H2D alone.)
    s_in, s_run, s_out = (torch.cuda.Stream(device=dev) for _ in range(3))
    bufs = []
    for _ in range(depth):
        bufs.append((torch.empty((chunk, n, w), dtype=torch.float64, device=dev),
                     torch.empty((chunk, n), dtype=torch.float64, device=dev),
                     torch.empty((chunk, n, w), dtype=torch.float64, device=dev),
                     torch.empty(chunk, dtype=torch.float64, device=dev),
                     torch.empty(chunk, dtype=torch.float64, device=dev),
                     new_status(chunk, dev),
                     (Bands.empty(chunk, n, k, 0, 32, device=dev), Vecs.empty(chunk, n, 32, device=dev),
                      Bands.empty(chunk, n, k, 0, 32, device=dev)) if tile == 32 else None))
    cur = torch.cuda.current_stream(dev)
    for st_ in (s_in, s_run, s_out):
        st_.wait_stream(cur)
    in_free = [None] * depth   # the chunk's inputs have been consumed by the kernels
    out_free = [None] * depth  # the chunk's outputs have left the device
    for ci, a in enumerate(range(0, B, chunk)):
        b = min(B, a + chunk)
        m = b - a
        slot = ci % depth
        dL, dy, dLb, dloss, dtb, st, t32 = bufs[slot]
        with torch.cuda.stream(s_in):
            if in_free[slot] is not None:
                s_in.wait_event(in_free[slot])
            dL[:m].copy_(L_host[a:b], non_blocking=True)
            dy[:m].copy_(y_host[a:b], non_blocking=True)
            ev_in = torch.cuda.Event()
            ev_in.record(s_in)
        with torch.cuda.stream(s_run):
            s_run.wait_event(ev_in)
            if out_free[slot] is not None:
                s_run.wait_event(out_free[slot])
            Lb = Bands(dL[:m], m, n, k, 0, 1)
            Yv = Vecs(dy[:m], m, n, 1)
            Lbar = Bands(dLb[:m], m, n, k, 0, 1)
            if t32 is None:
                marginal_likelihood_grad(Lb, Yv, tau2, check=False, out=(dloss[:m], Lbar, dtb[:m], st))
            else:
                L32, y32, Lbar32 = (_prefix(x, m) for x in t32)
                Lb.to_tile(32, L32)
                Yv.to_tile(32, y32)
                marginal_likelihood_grad(L32, y32, tau2, check=False, out=(dloss[:m], Lbar32, dtb[:m], st))
                Lbar32.to_tile(1, Lbar)
            in_free[slot] = torch.cuda.Event()
            in_free[slot].record(s_run)
            ev_run = torch.cuda.Event()
            ev_run.record(s_run)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_run)
            lbar_h[a:b].copy_(dLb[:m], non_blocking=True)
            loss_h[a:b].copy_(dloss[:m], non_blocking=True)
            tbar_h[a:b].copy_(dtb[:m], non_blocking=True)
            out_free[slot] = torch.cuda.Event()
            out_free[slot].record(s_out)
    for st_ in (s_in, s_run, s_out):
        cur.wait_stream(st_)
    return loss_h, lbar_h, tbar_h


def _prefix(x, m):
    """The first m matrices of a tile-32 container (whole tiles + a partial one)."""
    t = (m + 31) // 32
    if isinstance(x, Bands):
        return Bands(x.data[:t], m, x.n, x.lower, x.upper, 32)
    return Vecs(x.data[:t], m, x.n, 32)
