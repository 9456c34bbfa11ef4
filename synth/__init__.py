"""Seeded synthetic input generators shared by the tests, smoke() and bench.py.

This module holds NONE of the method's arithmetic (no network, no target, no
gradient, no update, no sampler): it only produces the transitions and initial
parameters that both the CUDA path and the oracle consume, so both sides see the
same bytes. Recipes:

* G-uniform (parity): every byte of s and s' uniform in [0,255]; a uniform over
  |A|; r uniform in {-1, 0, +1}; terminal with p = 0.1.
* G-pong (throughput; "Pong-shaped" frames of BASELINE.json): background 87,
  two 4x16 paddles of value 147 at x = 8 and x = 72 with per-frame heights, a
  2x2 ball of value 236 moving linearly across the frames; s' is s shifted by
  one frame plus a new frame; a uniform over |A|; r = +-1 with p = 0.01 each,
  else 0; terminal with p = 1e-3.
* theta0: independent N(0, std_t^2) per tensor, tensor list supplied by the caller.
"""
from __future__ import annotations

from typing import Sequence, Tuple

import numpy as np


def g_uniform(n: int, frames: int, height: int, width: int, n_actions: int, seed: int):
    rng = np.random.Generator(np.random.PCG64(seed))
    s = rng.integers(0, 256, size=(n, frames, height, width), dtype=np.uint8)
    s_next = rng.integers(0, 256, size=(n, frames, height, width), dtype=np.uint8)
    a = rng.integers(0, n_actions, size=n, dtype=np.int32)
    r = rng.integers(-1, 2, size=n).astype(np.float32)
    term = (rng.random(n) < 0.1).astype(np.uint8)
    return s, a, r, s_next, term


def _pong_frames_np(n: int, nf: int, height: int, width: int, rng: np.random.Generator) -> np.ndarray:
    frames = np.full((n, nf, height, width), 87, np.uint8)
    pad_h, pad_w = min(16, height), min(4, width)
    ly0 = rng.integers(0, max(1, height - pad_h + 1), size=n)
    ry0 = rng.integers(0, max(1, height - pad_h + 1), size=n)
    ldy = rng.integers(-3, 4, size=n)
    rdy = rng.integers(-3, 4, size=n)
    bx0 = rng.integers(0, max(1, width - 1), size=n)
    by0 = rng.integers(0, max(1, height - 1), size=n)
    vx = rng.integers(-4, 5, size=n)
    vy = rng.integers(-4, 5, size=n)
    xl = min(8, max(0, width - pad_w))
    xr = min(72, max(0, width - pad_w))
    span_y = max(1, height - pad_h + 1)
    rows = np.arange(n)
    for f in range(nf):
        ly = (ly0 + f * ldy) % span_y
        ry = (ry0 + f * rdy) % span_y
        bx = (bx0 + f * vx) % max(1, width - 1)
        by = (by0 + f * vy) % max(1, height - 1)
        for dy in range(pad_h):
            frames[rows, f, ly + dy, xl:xl + pad_w] = 147
            frames[rows, f, ry + dy, xr:xr + pad_w] = 147
        for dy in range(min(2, height)):
            for dx in range(min(2, width)):
                frames[rows, f, by + dy, bx + dx] = 236
    return frames


def g_pong(n: int, frames: int, height: int, width: int, n_actions: int, seed: int):
    rng = np.random.Generator(np.random.PCG64(seed))
    fr = _pong_frames_np(n, frames + 1, height, width, rng)
    s = np.ascontiguousarray(fr[:, :frames])
    s_next = np.ascontiguousarray(fr[:, 1:])
    a = rng.integers(0, n_actions, size=n, dtype=np.int32)
    u = rng.random(n)
    r = np.where(u < 0.01, 1.0, np.where(u < 0.02, -1.0, 0.0)).astype(np.float32)
    term = (rng.random(n) < 1e-3).astype(np.uint8)
    return s, a, r, s_next, term


def g_pong_torch(n: int, frames: int, height: int, width: int, n_actions: int, seed: int, device):
    """G-pong generated with torch ops directly on `device` (bench prefill of 1M-slot replays)."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    nf = frames + 1
    pad_h, pad_w = min(16, height), min(4, width)
    span_y = max(1, height - pad_h + 1)

    def ri(lo, hi):
        return torch.randint(lo, hi, (n,), generator=g, device=device)

    ly0, ry0 = ri(0, span_y), ri(0, span_y)
    ldy, rdy = ri(-3, 4), ri(-3, 4)
    bx0, by0 = ri(0, max(1, width - 1)), ri(0, max(1, height - 1))
    vx, vy = ri(-4, 5), ri(-4, 5)
    f = torch.arange(nf, device=device).view(1, nf)
    ly = (ly0.view(n, 1) + f * ldy.view(n, 1)) % span_y
    ry = (ry0.view(n, 1) + f * rdy.view(n, 1)) % span_y
    bx = (bx0.view(n, 1) + f * vx.view(n, 1)) % max(1, width - 1)
    by = (by0.view(n, 1) + f * vy.view(n, 1)) % max(1, height - 1)
    yy = torch.arange(height, device=device).view(1, 1, height, 1)
    xx = torch.arange(width, device=device).view(1, 1, 1, width)
    xl = min(8, max(0, width - pad_w))
    xr = min(72, max(0, width - pad_w))
    lmask = (yy >= ly[..., None, None]) & (yy < ly[..., None, None] + pad_h) & (xx >= xl) & (xx < xl + pad_w)
    rmask = (yy >= ry[..., None, None]) & (yy < ry[..., None, None] + pad_h) & (xx >= xr) & (xx < xr + pad_w)
    bmask = (yy >= by[..., None, None]) & (yy < by[..., None, None] + 2) & (xx >= bx[..., None, None]) & (
        xx < bx[..., None, None] + 2)
    fr = torch.full((n, nf, height, width), 87, dtype=torch.uint8, device=device)
    fr[lmask | rmask] = 147
    fr[bmask] = 236
    s = fr[:, :frames].contiguous()
    s_next = fr[:, 1:].contiguous()
    a = torch.randint(0, n_actions, (n,), generator=g, device=device, dtype=torch.int32)
    u = torch.rand((n,), generator=g, device=device)
    r = torch.where(u < 0.01, 1.0, torch.where(u < 0.02, -1.0, 0.0)).to(torch.float32)
    term = (torch.rand((n,), generator=g, device=device) < 1e-3).to(torch.uint8)
    return s, a, r, s_next, term


def init_theta(tensors: Sequence[Tuple[int, int]], stds: Sequence[float], seed: int) -> np.ndarray:
    """theta0 as float32: tensor t = (offset, count) drawn N(0, stds[t]^2)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    P = max(o + c for o, c in tensors)
    th = np.zeros(P, np.float32)
    for (o, c), sd in zip(tensors, stds):
        th[o:o + c] = (rng.standard_normal(c) * sd).astype(np.float32)
    return th
