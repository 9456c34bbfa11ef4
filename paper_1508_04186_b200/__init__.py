"""Python binding of libdqn.so — the C ABI of include/dqn.h.

Argument marshalling only: every step of the hot path (sampling, gather,
convolutions, FC layers, TD head, backward, RMSProp shard update, NCCL
push/fetch) runs inside libdqn.so's CUDA kernels. There is no CPU or PyTorch
fallback: importing this package without the built library raises.

Names follow the paper (arXiv 1508.04186): theta, theta^ (target), n
(generation), b (minibatch), C (target_sync), n_push / n_fetch (Downpour).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence, Tuple

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libdqn.so")

OK, EINVAL, EEMPTY, ENONFINITE, ENOMEM, ECUDA, ENCCL, ESTATE = 0, -1, -2, -3, -4, -5, -6, -7
FP32, BF16 = 0, 1
DETERMINISTIC, ASYNC, ASYNC_LAG1 = 0, 1, 2
SERVER_MEAN, SERVER_PER_GRADIENT = 0, 1
PARAMS_SERVER, PARAMS_LOCAL, PARAMS_TARGET, PARAMS_GRAD, PARAMS_RMS = 0, 1, 2, 3, 4
PARAMS_LOCAL_BF16, PARAMS_TARGET_BF16 = 5, 6  # bf16 working copies widened to fp32 (diagnostic)
_NAMES = {0: "OK", -1: "EINVAL", -2: "EEMPTY", -3: "ENONFINITE", -4: "ENOMEM", -5: "ECUDA", -6: "ENCCL",
          -7: "ESTATE"}


class DqnError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_NAMES.get(code, code)}: {msg}")
        self.code = code


class _Config(C.Structure):
    _fields_ = [("frames", C.c_int32), ("height", C.c_int32), ("width", C.c_int32), ("n_conv", C.c_int32),
                ("conv_filters", C.c_int32 * 4), ("conv_kernel", C.c_int32 * 4), ("conv_stride", C.c_int32 * 4),
                ("n_fc", C.c_int32), ("fc_units", C.c_int32 * 4), ("n_actions", C.c_int32),
                ("minibatch", C.c_int32), ("gamma", C.c_double), ("lr", C.c_double), ("rms_decay", C.c_double),
                ("rms_eps", C.c_double), ("err_clip", C.c_double), ("replay_capacity", C.c_int64),
                ("n_push", C.c_int32), ("n_fetch", C.c_int32), ("target_sync", C.c_int64),
                ("precision", C.c_int32), ("sync_mode", C.c_int32), ("seed", C.c_uint64),
                ("init_std", C.c_double), ("init_seed", C.c_uint64), ("init_params", C.c_void_p),
                ("server_rule", C.c_int32), ("replay_dedup", C.c_int32), ("keep_grad", C.c_int32),
                ("replay_prio_alpha", C.c_double), ("replay_prio_eps", C.c_double)]


class _Stats(C.Structure):
    _fields_ = [("loss_mean", C.c_double), ("generation", C.c_int64), ("steps_done", C.c_int64),
                ("device_ms", C.c_float), ("nonfinite_elems", C.c_int64), ("sampled_idx", C.c_void_p),
                ("target_argmax", C.c_void_p), ("loss_per_step", C.c_void_p), ("kernel_launches", C.c_int64),
                ("staleness_hist", C.c_int64 * 32), ("step_generation", C.c_void_p), ("grad_ms", C.c_double),
                ("update_ms", C.c_double), ("comm_ms", C.c_double), ("td_error", C.c_void_p)]


class _CollectStats(C.Structure):
    _fields_ = [("env_steps", C.c_int64), ("episodes", C.c_int64), ("reward_sum", C.c_double), ("device_ms", C.c_float),
                ("actions", C.c_void_p), ("rewards", C.c_void_p), ("terminals", C.c_void_p)]


class _RegionTime(C.Structure):
    _fields_ = [("name", C.c_char * 48), ("avg_us", C.c_double), ("kernels", C.c_int32), ("steps", C.c_int32)]


@dataclass
class Config:
    """dqn_config (include/dqn.h). Defaults: Mnih-2013 DQN of BASELINE.json configs[0]."""
    frames: int = 4
    height: int = 84
    width: int = 84
    convs: Sequence[Tuple[int, int, int]] = ((16, 8, 4), (32, 4, 2))   # (filters, kernel, stride)
    fcs: Sequence[int] = (256,)
    n_actions: int = 6
    minibatch: int = 32
    gamma: float = 0.99
    lr: float = 2.5e-4
    rms_decay: float = 0.9
    rms_eps: float = 1e-8
    err_clip: float = 0.0
    replay_capacity: int = 1000
    n_push: int = 1
    n_fetch: int = 1
    target_sync: int = 2**62
    precision: int = FP32
    sync_mode: int = DETERMINISTIC
    seed: int = 0xD15EA5E
    init_std: float = 0.01
    init_seed: int = 7
    server_rule: int = 0   # SERVER_MEAN (A7) | SERVER_PER_GRADIENT (A33)
    replay_dedup: int = 0  # 1: F+1 frames per slot (s' = s shifted by one frame + a new frame)
    keep_grad: int = 0     # 1: the update kernels also store the pushed gradient (DQN_PARAMS_GRAD)
    replay_prio_alpha: float = 0.0  # prioritized replay (A41): 0 = uniform, 1 or 0.5
    replay_prio_eps: float = 0.0

    def to_c(self, init_ptr: Optional[int] = None) -> _Config:
        c = _Config()
        c.frames, c.height, c.width = self.frames, self.height, self.width
        c.n_conv = len(self.convs)
        for i, (f, k, s) in enumerate(self.convs):
            c.conv_filters[i], c.conv_kernel[i], c.conv_stride[i] = f, k, s
        c.n_fc = len(self.fcs)
        for i, u in enumerate(self.fcs):
            c.fc_units[i] = u
        for name in ("n_actions", "minibatch", "gamma", "lr", "rms_decay", "rms_eps", "err_clip", "replay_capacity",
                     "n_push", "n_fetch", "target_sync", "precision", "sync_mode", "seed", "init_std", "init_seed",
                     "server_rule", "replay_dedup", "keep_grad", "replay_prio_alpha", "replay_prio_eps"):
            setattr(c, name, getattr(self, name))
        c.init_params = init_ptr
        return c

    @property
    def state_shape(self):
        return (self.frames, self.height, self.width)


_lib = None


def lib() -> C.CDLL:
    """Load libdqn.so; raises if it has not been built (no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1508_04186_b200.build` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        L.dqn_param_count.restype = C.c_int64
        L.dqn_param_count.argtypes = [C.POINTER(_Config)]
        L.dqn_nccl_id_bytes.restype = C.c_int32
        L.dqn_nccl_unique_id.argtypes = [P]
        L.dqn_create.argtypes = [C.POINTER(_Config), C.c_int, C.c_int, P, P, C.POINTER(P)]
        L.dqn_push_transitions.argtypes = [P, C.c_int64, P, P, P, P, P]
        L.dqn_train_steps.argtypes = [P, C.c_int64, C.POINTER(_Stats)]
        L.dqn_store_and_train.argtypes = [P, C.c_int64, P, P, P, P, P, C.POINTER(_Stats)]
        L.dqn_q_values.argtypes = [P, C.c_int64, P, P, P]
        L.dqn_profile_steps.argtypes = [P, C.c_int64, C.POINTER(_RegionTime), C.c_int32, C.POINTER(C.c_int32)]
        L.dqn_get_params.argtypes = [P, C.c_int, P, C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_uint64)]
        L.dqn_replay_size.argtypes = [P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.dqn_get_priorities.argtypes = [P, P, C.c_int64, P]
        L.dqn_last_error.restype = C.c_char_p
        L.dqn_last_error.argtypes = [P]
        L.dqn_destroy.argtypes = [P]
        L.dqn_collect.argtypes = [P, C.c_int32, C.c_int32, C.c_int64, C.c_double, C.c_uint64, C.POINTER(_CollectStats)]
        L.dqn_env_stacks.argtypes = [P, P, C.c_int64]
        _lib = L
    return _lib


EXPORTED = ("dqn_param_count", "dqn_nccl_id_bytes", "dqn_nccl_unique_id", "dqn_create", "dqn_push_transitions",
            "dqn_train_steps", "dqn_profile_steps", "dqn_q_values", "dqn_get_params", "dqn_replay_size", "dqn_last_error",
            "dqn_destroy", "dqn_collect", "dqn_env_stacks", "dqn_store_and_train", "dqn_get_priorities")


def param_count(cfg: Config) -> int:
    return int(lib().dqn_param_count(C.byref(cfg.to_c())))


def nccl_unique_id() -> bytes:
    n = lib().dqn_nccl_id_bytes()
    buf = C.create_string_buffer(n)
    rc = lib().dqn_nccl_unique_id(buf)
    if rc:
        raise DqnError(rc, "ncclGetUniqueId failed")
    return buf.raw


def _ptr(x, dtype) -> Tuple[int, object]:
    """(address, keep-alive) of a contiguous numpy array or torch tensor (host or CUDA)."""
    if x is None:
        return None, None
    try:
        import torch
        if isinstance(x, torch.Tensor):
            t = x.contiguous()
            want = {np.uint8: torch.uint8, np.int32: torch.int32, np.float32: torch.float32}[dtype]
            if t.dtype != want:
                t = t.to(want)
            return t.data_ptr(), t
    except ImportError:
        pass
    a = np.ascontiguousarray(x, dtype=dtype)
    return a.ctypes.data, a


def _out_ptr(x, dtype, name: str) -> Tuple[int, object]:
    """Address of an output buffer the library writes in place: it must already be contiguous with the
    right dtype (a converted copy would be written instead of the caller's buffer)."""
    try:
        import torch
        if isinstance(x, torch.Tensor):
            want = {np.int32: torch.int32, np.float32: torch.float32}[dtype]
            if x.dtype != want or not x.is_contiguous():
                raise ValueError(f"{name} must be a contiguous {want} tensor")
            return x.data_ptr(), x
    except ImportError:
        pass
    if not isinstance(x, np.ndarray) or x.dtype != dtype or not x.flags["C_CONTIGUOUS"]:
        raise ValueError(f"{name} must be a C-contiguous numpy array of {np.dtype(dtype).name}")
    return x.ctypes.data, x


class DQN:
    """One replica + parameter-server shard on the current CUDA device (dqn_ctx)."""

    def __init__(self, cfg: Config, rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None,
                 stream: Optional[int] = None, init_params=None):
        self.cfg = cfg
        L = lib()
        ip, keep = _ptr(init_params, np.float32)
        c = cfg.to_c(ip)
        h = C.c_void_p()
        idbuf = C.create_string_buffer(nccl_id, len(nccl_id)) if nccl_id is not None else None
        rc = L.dqn_create(C.byref(c), rank, world, idbuf, stream, C.byref(h))
        if rc:
            raise DqnError(rc, L.dqn_last_error(None).decode())
        self._h = h
        self.P = param_count(cfg)
        del keep

    def _check(self, rc: int):
        if rc:
            raise DqnError(rc, lib().dqn_last_error(self._h).decode())

    def push(self, s, a, r, s_next, term) -> None:
        n = len(a)
        ps, k1 = _ptr(s, np.uint8)
        pa, k2 = _ptr(a, np.int32)
        pr, k3 = _ptr(r, np.float32)
        pn, k4 = _ptr(s_next, np.uint8)
        pt, k5 = _ptr(term, np.uint8)
        self._check(lib().dqn_push_transitions(self._h, n, ps, pa, pr, pn, pt))

    def train(self, k: int, want_idx: bool = False, want_argmax: bool = False, want_loss: bool = False,
              store=None, want_generation: bool = False, want_delta: bool = False) -> dict:
        """k replica steps (dqn_train_steps); with store = (s, a, r, s_next, term) of k transitions, Alg. 1's
        loop instead: transition i is stored, then step i runs (dqn_store_and_train)."""
        st = _Stats()
        b = self.cfg.minibatch
        idx = np.zeros((k, b), np.int32) if want_idx else None
        am = np.zeros((k, b), np.int32) if want_argmax else None
        lp = np.zeros(k, np.float32) if want_loss else None
        sg = np.zeros(k, np.int64) if want_generation else None
        dl = np.zeros((k, b), np.float32) if want_delta else None
        st.td_error = dl.ctypes.data if dl is not None else None
        st.step_generation = sg.ctypes.data if sg is not None else None
        st.sampled_idx = idx.ctypes.data if idx is not None else None
        st.target_argmax = am.ctypes.data if am is not None else None
        st.loss_per_step = lp.ctypes.data if lp is not None else None
        if store is None:
            rc = lib().dqn_train_steps(self._h, k, C.byref(st))
        else:
            s_, a_, r_, sn_, t_ = store
            if len(a_) != k:
                raise ValueError("store needs exactly k transitions")
            ps, k1 = _ptr(s_, np.uint8)
            pa, k2 = _ptr(a_, np.int32)
            pr, k3 = _ptr(r_, np.float32)
            pn, k4 = _ptr(sn_, np.uint8)
            pt, k5 = _ptr(t_, np.uint8)
            rc = lib().dqn_store_and_train(self._h, k, ps, pa, pr, pn, pt, C.byref(st))
        out = dict(loss_mean=st.loss_mean, generation=st.generation, steps_done=st.steps_done,
                   device_ms=st.device_ms, nonfinite_elems=st.nonfinite_elems, idx=idx, argmax=am, loss=lp,
                   kernel_launches=st.kernel_launches, staleness=np.array(st.staleness_hist[:], np.int64), rc=rc,
                   step_generation=sg, grad_ms=st.grad_ms, update_ms=st.update_ms, comm_ms=st.comm_ms, delta=dl)
        self._check(rc)
        return out

    def collect(self, n_envs: int, grid: int, steps: int, epsilon: float, seed: int, want_log: bool = False) -> dict:
        """NEXT-3: `steps` acting steps of n_envs on-GPU Snake games with the eps-greedy policy on theta_local;
        every transition is stored into the replay. Returns stats (+ per-step logs [steps][n_envs])."""
        st = _CollectStats()
        logs = {}
        if want_log:
            logs = dict(a=np.zeros((steps, n_envs), np.int32), r=np.zeros((steps, n_envs), np.float32),
                        term=np.zeros((steps, n_envs), np.uint8))
            st.actions, st.rewards, st.terminals = (logs["a"].ctypes.data, logs["r"].ctypes.data,
                                                    logs["term"].ctypes.data)
        self._check(lib().dqn_collect(self._h, n_envs, grid, steps, epsilon, seed, C.byref(st)))
        return dict(env_steps=st.env_steps, episodes=st.episodes, reward_sum=st.reward_sum, device_ms=st.device_ms,
                    **logs)

    def env_stacks(self, n_envs: int) -> np.ndarray:
        c = self.cfg
        out = np.zeros((n_envs, c.frames, c.height, c.width), np.uint8)
        self._check(lib().dqn_env_stacks(self._h, out.ctypes.data, out.nbytes))
        return out

    def profile(self, k: int) -> list:
        """k real steps with CUDA events around every region of the step graph -> per-region mean us."""
        buf = (_RegionTime * 64)()
        n = C.c_int32()
        self._check(lib().dqn_profile_steps(self._h, k, buf, 64, C.byref(n)))
        return [dict(name=buf[i].name.decode(), avg_us=buf[i].avg_us, kernels=buf[i].kernels, steps=buf[i].steps)
                for i in range(min(n.value, 64))]

    def q_values(self, states, q_out=None, argmax_out=None):
        """Q(s, .; theta_local) and the greedy actions (dqn_q_values). Caller-given outputs must be contiguous
        float32 / int32 (numpy or torch, host or CUDA): they are written in place."""
        n = len(states)
        A = self.cfg.n_actions
        ps, k1 = _ptr(states, np.uint8)
        q = q_out if q_out is not None else np.zeros((n, A), np.float32)
        am = argmax_out if argmax_out is not None else np.zeros(n, np.int32)
        pq, kq = _out_ptr(q, np.float32, "q_out")
        pa, ka = _out_ptr(am, np.int32, "argmax_out")
        self._check(lib().dqn_q_values(self._h, n, ps, pq, pa))
        del k1, kq, ka
        return q, am

    def params(self, which: int = PARAMS_SERVER, out=None):
        o = out if out is not None else np.zeros(self.P, np.float32)
        po, ko = _out_ptr(o, np.float32, "out")
        n = C.c_int64()
        g = C.c_uint64()
        self._check(lib().dqn_get_params(self._h, which, po, self.P, C.byref(n), C.byref(g)))
        return o

    def generation(self, which: int = PARAMS_SERVER) -> int:
        n = C.c_int64()
        g = C.c_uint64()
        self._check(lib().dqn_get_params(self._h, which, None, 0, C.byref(n), C.byref(g)))
        return int(g.value)

    def priorities(self) -> Tuple[np.ndarray, float]:
        """Prioritized replay (A41): the leaf priorities [replay_capacity] and the sum-tree total."""
        out = np.zeros(self.cfg.replay_capacity, np.float32)
        tot = np.zeros(1, np.float32)
        self._check(lib().dqn_get_priorities(self._h, out.ctypes.data, out.size, tot.ctypes.data))
        return out, float(tot[0])

    def replay_size(self) -> Tuple[int, int]:
        c, s = C.c_int64(), C.c_int64()
        self._check(lib().dqn_replay_size(self._h, C.byref(c), C.byref(s)))
        return int(c.value), int(s.value)

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().dqn_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
