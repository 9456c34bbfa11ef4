"""ctypes wrapper of the fp64 CPU oracle (oracle/dqn_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / ``--impl reference`` legs of bench.py. The product package
(paper_1508_04186_b200) never imports this module, and this module imports
nothing from the product package.

Every wrapped function cites its passage in dqn_oracle.c; readings of the paper
are DESIGN.md §3 (A1..A29).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dqn_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile the oracle with plain IEEE semantics (no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "dqn_oracle.h"))
    ):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-fopenmp", "-shared", "-fPIC",
               "-o", _LIB_PATH + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB_PATH + ".tmp", _LIB_PATH)
    return _LIB_PATH


class _Net(C.Structure):
    _fields_ = [("frames", C.c_int32), ("height", C.c_int32), ("width", C.c_int32),
                ("n_conv", C.c_int32), ("conv_filters", C.c_int32 * 4), ("conv_kernel", C.c_int32 * 4),
                ("conv_stride", C.c_int32 * 4), ("n_fc", C.c_int32), ("fc_units", C.c_int32 * 4),
                ("n_actions", C.c_int32)]


class _Cfg(C.Structure):
    _fields_ = [("n_replicas", C.c_int32), ("minibatch", C.c_int32), ("n_push", C.c_int32),
                ("n_fetch", C.c_int32), ("target_sync", C.c_int64), ("gamma", C.c_double),
                ("lr", C.c_double), ("rms_decay", C.c_double), ("rms_eps", C.c_double),
                ("err_clip", C.c_double), ("seed", C.c_uint64), ("fetch_lag", C.c_int32), ("server_rule", C.c_int32),
                ("fetch_gen", C.c_void_p)]


@dataclass
class Net:
    """Network shape (App. A; layer lists from BASELINE.json configs, A16)."""
    frames: int = 4
    height: int = 84
    width: int = 84
    convs: Sequence[tuple] = ((16, 8, 4), (32, 4, 2))  # (filters, kernel, stride)
    fcs: Sequence[int] = (256,)
    n_actions: int = 6

    def c(self) -> _Net:
        n = _Net()
        n.frames, n.height, n.width = self.frames, self.height, self.width
        n.n_conv = len(self.convs)
        for i, (f, k, s) in enumerate(self.convs):
            n.conv_filters[i], n.conv_kernel[i], n.conv_stride[i] = f, k, s
        n.n_fc = len(self.fcs)
        for i, u in enumerate(self.fcs):
            n.fc_units[i] = u
        n.n_actions = self.n_actions
        return n

    @property
    def state_size(self) -> int:
        return self.frames * self.height * self.width


MNIH = Net()
NATURE_SCALED = Net(convs=((32, 8, 4), (64, 4, 2), (64, 3, 1)), fcs=(512,), n_actions=18)


@dataclass
class TrainCfg:
    n_replicas: int = 1
    minibatch: int = 32
    n_push: int = 1
    n_fetch: int = 1
    target_sync: int = 2**62
    gamma: float = 0.99
    lr: float = 2.5e-4
    rms_decay: float = 0.9
    rms_eps: float = 1e-8
    err_clip: float = 0.0
    seed: int = 0xD15EA5E
    fetch_lag: int = 0   # O13 / A32: a fetch returns theta as it was `fetch_lag` rounds ago
    server_rule: int = 0  # 0: mean per round (A7); 1: Alg. 2 literally, one update per gradient (A33)
    fetch_gen: Optional[np.ndarray] = None  # [N][n_fetches] generation of every fetch (realised async schedule, A40)

    def c(self) -> _Cfg:
        c = _Cfg()
        for f, _ in _Cfg._fields_:
            if f != "fetch_gen":
                setattr(c, f, getattr(self, f))
        if self.fetch_gen is not None:
            c._keep = np.ascontiguousarray(self.fetch_gen, np.int64)  # alive as long as the struct
            c.fetch_gen = c._keep.ctypes.data
        return c


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        D = C.POINTER(C.c_double)
        U8 = C.POINTER(C.c_uint8)
        I32 = C.POINTER(C.c_int32)
        I64 = C.POINTER(C.c_int64)
        _lib.or_threads.restype = C.c_int32
        _lib.or_set_threads.argtypes = [C.c_int32]
        _lib.or_param_count.restype = C.c_int64
        _lib.or_param_count.argtypes = [C.POINTER(_Net)]
        _lib.or_tensor_table.restype = C.c_int32
        _lib.or_tensor_table.argtypes = [C.POINTER(_Net), I64, I64, C.c_int32]
        _lib.or_philox4x32_10.argtypes = [C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        _lib.or_sample_index.restype = C.c_int64
        _lib.or_sample_index.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint32, C.c_int64]
        _lib.or_conv_forward.argtypes = [D, C.c_int, C.c_int, C.c_int, D, D, C.c_int, C.c_int, C.c_int, D]
        _lib.or_fc_forward.argtypes = [D, C.c_int, D, D, C.c_int, D]
        _lib.or_forward.argtypes = [C.POINTER(_Net), D, D, D]
        _lib.or_q_values.argtypes = [C.POINTER(_Net), D, C.c_int64, U8, D, I32]
        _lib.or_targets.argtypes = [C.POINTER(_Net), D, C.c_int, U8, D, U8, C.c_double, D, I32]
        _lib.or_loss_grad.restype = C.c_double
        _lib.or_loss_grad.argtypes = [C.POINTER(_Net), D, C.c_int, U8, I32, D, C.c_double, D]
        _lib.or_loss_grad_x.restype = C.c_double
        _lib.or_loss_grad_x.argtypes = [C.POINTER(_Net), D, C.c_int, D, I32, D, C.c_double, D]
        _lib.or_min_abs_preact.restype = C.c_double
        _lib.or_min_abs_preact.argtypes = [C.POINTER(_Net), D, C.c_int64, U8]
        _lib.or_rmsprop.argtypes = [D, D, D, C.c_int64, C.c_double, C.c_double, C.c_double]
        _lib.or_snake_reset.argtypes = [C.POINTER(Snake), C.c_int, C.c_uint64, C.c_uint32, C.c_uint64]
        _lib.or_snake_step.restype = C.c_double
        _lib.or_snake_step.argtypes = [C.POINTER(Snake), C.c_int, C.c_int, C.c_uint64, C.c_uint32, C.c_uint64,
                                       C.POINTER(C.c_int)]
        _lib.or_snake_render.argtypes = [C.POINTER(Snake), C.c_int, C.c_int, U8]
        _lib.or_eps_greedy.restype = C.c_int
        _lib.or_eps_greedy.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, C.c_int]
        _lib.or_collect.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int64, C.c_uint64, C.c_uint64, I32,
                                    C.c_int, C.POINTER(Snake), U8, C.c_uint64, I32, D, U8, I64]
        _lib.or_run.restype = C.c_int
        _lib.or_run.argtypes = [C.POINTER(_Net), C.POINTER(_Cfg), C.c_int64, I64, C.POINTER(U8), C.POINTER(I32),
                                C.POINTER(D), C.POINTER(U8), C.POINTER(U8), D, C.c_int64, D, D, I64, D, I64, I32, D, I64]
    return _lib


class Snake(C.Structure):
    """or_snake: body length, direction, apple cell, steps since the last apple, body cells head first."""
    _fields_ = [("len", C.c_int32), ("dir", C.c_int32), ("apple", C.c_int32), ("since", C.c_int32),
                ("body", C.c_int16 * 1024)]


def eps_threshold(eps: float) -> int:
    """floor(eps * 2^32) in [0, 2^32]: explore iff the 32-bit draw is below it."""
    return min(1 << 32, int(math.floor(eps * 4294967296.0)))


def snake_reset(n: int, seed: int, env: int, t: int) -> Snake:
    g = Snake()
    lib().or_snake_reset(C.byref(g), n, seed, env, t)
    return g


def snake_step(g: Snake, n: int, action: int, seed: int, env: int, t: int):
    term = C.c_int(0)
    r = lib().or_snake_step(C.byref(g), n, action, seed, env, t, C.byref(term))
    return r, bool(term.value)


def snake_render(g: Snake, n: int, px: int) -> np.ndarray:
    f = np.zeros((n * px, n * px), np.uint8)
    lib().or_snake_render(C.byref(g), n, px, _p(f, C.c_uint8))
    return f


def eps_greedy(seed: int, env: int, t: int, eps: float, greedy: int) -> int:
    return int(lib().or_eps_greedy(seed, env, t, eps_threshold(eps), greedy))


def collect(n: int, F: int, H: int, E: int, steps: int, seed: int, eps: float, greedy=None, state=None, t0: int = 0):
    """E Snake games x `steps` eps-greedy acting steps (or_collect). state = (games, stacks) to continue a
    previous call (else the initial resets). Returns dict(stacks, games, a, r, term, episodes)."""
    init = state is None
    games = (Snake * E)() if init else state[0]
    stacks = np.zeros((E, F, H, H), np.uint8) if init else state[1]
    a = np.zeros((steps, E), np.int32)
    r = np.zeros((steps, E), np.float64)
    t = np.zeros((steps, E), np.uint8)
    ep = np.zeros(E, np.int64)
    gr = None if greedy is None else np.ascontiguousarray(greedy, dtype=np.int32)
    lib().or_collect(n, F, H, E, steps, seed, eps_threshold(eps), _p(gr, C.c_int32) if gr is not None else None,
                     int(init), games, _p(stacks, C.c_uint8), t0, _p(a, C.c_int32), _p(r, C.c_double),
                     _p(t, C.c_uint8), _p(ep, C.c_int64))
    return dict(stacks=stacks, games=games, a=a, r=r, term=t, episodes=ep)


def _p(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def threads() -> int:
    """Threads the oracle's per-sample loops use (its results do not depend on it)."""
    return int(lib().or_threads())


def set_threads(n: int) -> None:
    """n <= 0: all host cores."""
    lib().or_set_threads(n)


def param_count(net: Net) -> int:
    return int(lib().or_param_count(C.byref(net.c())))


def tensor_table(net: Net):
    offs = np.zeros(32, np.int64)
    cnts = np.zeros(32, np.int64)
    t = lib().or_tensor_table(C.byref(net.c()), _p(offs, C.c_int64), _p(cnts, C.c_int64), 32)
    if t < 0:
        raise ValueError("invalid network")
    return list(zip(offs[:t].tolist(), cnts[:t].tolist()))


def philox4x32_10(ctr, key) -> List[int]:
    c = (C.c_uint32 * 4)(*ctr)
    k = (C.c_uint32 * 2)(*key)
    o = (C.c_uint32 * 4)()
    lib().or_philox4x32_10(c, k, o)
    return list(o)


def sample_index(seed: int, rank: int, T: int, j: int, size: int) -> int:
    return int(lib().or_sample_index(seed, rank, T, j, size))


def conv_forward(x: np.ndarray, w: np.ndarray, b: np.ndarray, stride: int) -> np.ndarray:
    x, w, b = _f64(x), _f64(w), _f64(b)
    Cc, H, W = x.shape
    N, C2, k, _ = w.shape
    assert C2 == Cc
    Ho, Wo = (H - k) // stride + 1, (W - k) // stride + 1
    out = np.zeros((N, Ho, Wo))
    lib().or_conv_forward(_p(x, C.c_double), Cc, H, W, _p(w, C.c_double), _p(b, C.c_double), N, k, stride,
                          _p(out, C.c_double))
    return out


def fc_forward(x: np.ndarray, w: np.ndarray, b: np.ndarray) -> np.ndarray:
    x, w, b = _f64(x), _f64(w), _f64(b)
    H, D = w.shape
    out = np.zeros(H)
    lib().or_fc_forward(_p(x, C.c_double), D, _p(w, C.c_double), _p(b, C.c_double), H, _p(out, C.c_double))
    return out


def forward(net: Net, theta: np.ndarray, x: np.ndarray) -> np.ndarray:
    theta, x = _f64(theta), _f64(x)
    q = np.zeros(net.n_actions)
    lib().or_forward(C.byref(net.c()), _p(theta, C.c_double), _p(x, C.c_double), _p(q, C.c_double))
    return q


def q_values(net: Net, theta: np.ndarray, states: np.ndarray):
    theta = _f64(theta)
    states = np.ascontiguousarray(states, dtype=np.uint8)
    n = states.shape[0]
    q = np.zeros((n, net.n_actions))
    am = np.zeros(n, np.int32)
    lib().or_q_values(C.byref(net.c()), _p(theta, C.c_double), n, _p(states, C.c_uint8), _p(q, C.c_double),
                      _p(am, C.c_int32))
    return q, am


def min_abs_preact(net: Net, theta: np.ndarray, states: np.ndarray) -> float:
    theta = _f64(theta)
    states = np.ascontiguousarray(states, dtype=np.uint8)
    return float(lib().or_min_abs_preact(C.byref(net.c()), _p(theta, C.c_double), states.shape[0],
                                         _p(states, C.c_uint8)))


def targets(net: Net, theta_hat: np.ndarray, s_next: np.ndarray, r, term, gamma: float):
    theta_hat = _f64(theta_hat)
    s_next = np.ascontiguousarray(s_next, dtype=np.uint8)
    r = _f64(r)
    term = np.ascontiguousarray(term, dtype=np.uint8)
    b = s_next.shape[0]
    y = np.zeros(b)
    am = np.zeros(b, np.int32)
    lib().or_targets(C.byref(net.c()), _p(theta_hat, C.c_double), b, _p(s_next, C.c_uint8), _p(r, C.c_double),
                     _p(term, C.c_uint8), gamma, _p(y, C.c_double), _p(am, C.c_int32))
    return y, am


def loss_grad(net: Net, theta, s, a, y, err_clip: float = 0.0):
    theta = _f64(theta)
    s = np.ascontiguousarray(s, dtype=np.uint8)
    a = np.ascontiguousarray(a, dtype=np.int32)
    y = _f64(y)
    g = np.zeros_like(theta)
    loss = lib().or_loss_grad(C.byref(net.c()), _p(theta, C.c_double), s.shape[0], _p(s, C.c_uint8),
                              _p(a, C.c_int32), _p(y, C.c_double), err_clip, _p(g, C.c_double))
    return loss, g


def loss_grad_x(net: Net, theta, x, a, y, err_clip: float = 0.0):
    theta, x, y = _f64(theta), _f64(x), _f64(y)
    a = np.ascontiguousarray(a, dtype=np.int32)
    g = np.zeros_like(theta)
    loss = lib().or_loss_grad_x(C.byref(net.c()), _p(theta, C.c_double), x.shape[0], _p(x, C.c_double),
                                _p(a, C.c_int32), _p(y, C.c_double), err_clip, _p(g, C.c_double))
    return loss, g


def rmsprop(theta, r, g, alpha: float, rho: float = 0.9, eps: float = 1e-8):
    theta, r, g = _f64(theta).copy(), _f64(r).copy(), _f64(g)
    lib().or_rmsprop(_p(theta, C.c_double), _p(r, C.c_double), _p(g, C.c_double), theta.size, alpha, rho, eps)
    return theta, r


@dataclass
class Replay:
    """One replica's pushes in push order (oldest first)."""
    s: np.ndarray        # [n, F, H, W] u8
    a: np.ndarray        # [n] int
    r: np.ndarray        # [n] float
    s_next: np.ndarray   # [n, F, H, W] u8
    term: np.ndarray     # [n] u8/bool


def run(net: Net, cfg: TrainCfg, capacity: int, replays: Sequence[Replay], theta0: np.ndarray, steps: int,
        want_grad0: bool = False) -> dict:
    """Alg. 1 x N workers + Alg. 2 server in lock-step (O2-O12)."""
    N = cfg.n_replicas
    assert len(replays) == N
    P = param_count(net)
    theta0 = _f64(theta0)
    assert theta0.size == P
    keep = []
    n_pushed = np.array([len(rp.a) for rp in replays], np.int64)
    S = (C.POINTER(C.c_uint8) * N)()
    SN = (C.POINTER(C.c_uint8) * N)()
    A = (C.POINTER(C.c_int32) * N)()
    R = (C.POINTER(C.c_double) * N)()
    TT = (C.POINTER(C.c_uint8) * N)()
    for k, rp in enumerate(replays):
        s = np.ascontiguousarray(rp.s, np.uint8)
        sn = np.ascontiguousarray(rp.s_next, np.uint8)
        a = np.ascontiguousarray(rp.a, np.int32)
        r = _f64(rp.r)
        t = np.ascontiguousarray(rp.term, np.uint8)
        keep += [s, sn, a, r, t]
        S[k], SN[k], A[k], R[k], TT[k] = (_p(s, C.c_uint8), _p(sn, C.c_uint8), _p(a, C.c_int32),
                                          _p(r, C.c_double), _p(t, C.c_uint8))
    theta = np.zeros(P)
    rr = np.zeros(P)
    n_out = np.zeros(1, np.int64)
    loss = np.zeros((N, steps))
    idx = np.zeros((N, steps, cfg.minibatch), np.int64)
    amax = np.zeros((N, steps, cfg.minibatch), np.int32)
    g0 = np.zeros(P) if want_grad0 else None
    stale = np.zeros(32, np.int64)
    rc = lib().or_run(C.byref(net.c()), C.byref(cfg.c()), capacity, _p(n_pushed, C.c_int64), S, A, R, SN, TT,
                      _p(theta0, C.c_double), steps, _p(theta, C.c_double), _p(rr, C.c_double),
                      _p(n_out, C.c_int64), _p(loss, C.c_double), _p(idx, C.c_int64), _p(amax, C.c_int32),
                      _p(g0, C.c_double) if g0 is not None else None, _p(stale, C.c_int64))
    return dict(rc=rc, theta=theta, r=rr, n=int(n_out[0]), loss=loss, idx=idx, amax=amax, grad0=g0,
                staleness=stale)
