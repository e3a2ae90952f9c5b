"""paper_2112_00364_b200 — B200-native SMC over PCFGs (arXiv 2112.00364).

Thin ctypes binding of ``libsmc.so`` (C ABI in ``include/smc.h``).  Every step
of the hot path runs in the CUDA kernels behind that ABI; this module only
marshals arguments.  There is NO CPU fallback: importing the package fails
loudly when the library is missing, and creating a handle fails without a
CUDA device.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libsmc.so")

if not os.path.exists(_LIB_PATH):
    raise ImportError(
        f"{_LIB_PATH} is missing: build it with `python paper_2112_00364_b200/csrc/build.py` "
        "(nvcc, sm_100a).  There is no CPU fallback.")

_lib = C.CDLL(_LIB_PATH, mode=C.RTLD_GLOBAL)

# ---- enums (include/smc.h) --------------------------------------------------
OK, EINVAL, ECUDA, ENCCL, EREJECTED, ENAN, EOVERFLOW, ESTATE = range(8)
CRBD, CLADS2, SEIR, GEOMETRIC, SSM, CONSTW, FIG3, STACKF, RESAMPLE_BENCH = 1, 2, 3, 10, 11, 12, 13, 14, 20
FLAG_STRICT = 1
FLAG_LINEAGE_RNG = 2
FLAG_ANALYTIC_UNDETECTED = 4
FLAG_INPLACE = 8

FIELDS = {
    CRBD: ["pc", "branch", "lambda", "mu"],
    CLADS2: ["pc", "branch", "sp", "sigma", "alpha", "eps", "lam"] + [f"pend{i}" for i in range(6)],
    SEIR: ["pc", "t", "lam_h", "del_h", "gam_h", "lam_m", "del_m", "rho",
           "sh", "eh", "ih", "rh", "sm", "em", "im"],
    GEOMETRIC: ["pc", "n"],
    SSM: ["pc", "t", "x"],
    CONSTW: ["pc", "k"],
    FIG3: ["pc", "n", "x"],
}


class smc_model(C.Structure):
    _fields_ = [("kind", C.c_int32), ("state_bytes", C.c_uint32),
                ("data", C.POINTER(C.c_double)), ("data_len", C.c_uint64),
                ("params", C.POINTER(C.c_double)), ("n_params", C.c_int32),
                ("flags", C.c_uint32)]


class smc_stats_t(C.Structure):
    _fields_ = [("n_total", C.c_uint64), ("n_local", C.c_uint64), ("epochs", C.c_uint64),
                ("resamples", C.c_uint64), ("alive_particle_steps", C.c_uint64),
                ("overflow", C.c_uint64), ("first_error_particle", C.c_int64),
                ("status", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32),
                ("shards", C.c_int32), ("state_bytes", C.c_uint32), ("done", C.c_uint32),
                ("draws", C.c_uint64), ("ms_propagate", C.c_double), ("ms_resample", C.c_double),
                ("timed_epochs", C.c_uint64), ("side_roots", C.c_uint64),
                ("max_rounds", C.c_uint32), ("max_side_nodes", C.c_uint32),
                ("distinct", C.c_uint64), ("ms_kernel", C.c_double * 4),
                ("stack_planes", C.c_uint64), ("guard_kills", C.c_uint64),
                ("deferred_gather", C.c_uint32),
                ("reserved0", C.c_uint32)]


ALLGATHER_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p)


class smc_comm(C.Structure):
    _fields_ = [("nccl_id", C.c_void_p), ("allgather", ALLGATHER_CB), ("user", C.c_void_p)]


H = C.c_void_p
_sig = {
    "smc_abi_version": ([], C.c_int),
    "smc_draw_peak": ([C.c_uint32, C.POINTER(C.c_double)], C.c_int),
    "smc_create": ([C.POINTER(smc_model), C.c_uint64, C.c_uint64], H),
    "smc_create_virtual": ([C.POINTER(smc_model), C.c_uint64, C.c_uint64, C.c_int32], H),
    "smc_create_sharded": ([C.POINTER(smc_model), C.c_uint64, C.c_uint64, C.c_int32, C.c_int32,
                            C.POINTER(smc_comm)], H),
    "smc_ipc_export": ([H, C.c_void_p], C.c_int),
    "smc_ipc_blob_bytes": ([], C.c_uint64),
    "smc_ipc_import": ([H, C.c_void_p], C.c_int),
    "smc_get_nccl_id": ([C.c_void_p], C.c_int),
    "smc_destroy": ([H], None),
    "smc_set_stream": ([H, C.c_void_p], C.c_int),
    "smc_reset": ([H, C.c_uint64], C.c_int),
    "smc_set_timing": ([H, C.c_int32], C.c_int),
    "smc_set_graph": ([H, C.c_int32], C.c_int),
    "smc_set_ess_threshold": ([H, C.c_uint32, C.c_uint32], C.c_int),
    "smc_set_data": ([H, C.POINTER(C.c_double), C.c_uint64], C.c_int),
    "smc_run": ([H], C.c_int),
    "smc_step": ([H, C.POINTER(C.c_int32)], C.c_int),
    "smc_log_z": ([H], C.c_double),
    "smc_ancestors": ([H, C.POINTER(C.c_uint32), C.c_uint64], C.c_int),
    "smc_log_weights": ([H, C.POINTER(C.c_double), C.c_uint64], C.c_int),
    "smc_state": ([H, C.c_void_p, C.c_uint64], C.c_int),
    "smc_nfields": ([H], C.c_int),
    "smc_fields": ([H, C.POINTER(C.c_double), C.c_uint64], C.c_int),
    "smc_stats": ([H, C.POINTER(smc_stats_t)], C.c_int),
    "smc_errmsg": ([H], C.c_char_p),
    "smc_resample_device": ([H, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32,
                             C.POINTER(C.c_double)], C.c_int),
    "smc_resample_host": ([H, C.POINTER(C.c_double), C.c_void_p, C.c_void_p,
                           C.POINTER(C.c_uint32), C.c_uint32, C.POINTER(C.c_double)], C.c_int),
    "smc_last_distinct": ([H, C.POINTER(C.c_uint64)], C.c_int),
    "smc_resample_grid": ([H, C.POINTER(C.c_int32)], C.c_int),
    "smc_load": ([H, C.c_void_p, C.c_void_p, C.c_int32], C.c_int),
    "smc_resample_step": ([H, C.c_uint32], C.c_int),
    "smc_plan_ranges": ([C.POINTER(C.c_uint64), C.c_int32, C.c_uint64, C.c_uint64,
                         C.POINTER(C.c_uint64)], C.c_int),
}
for _name, (_args, _res) in _sig.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res

EXPORTED = sorted(_sig)


class SmcError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"smc status {code}: {msg}")
        self.code = code


def _check(h, rc):
    if rc != OK:
        raise SmcError(rc, _lib.smc_errmsg(h).decode())
    return rc


def _stream_ptr(stream):
    """torch.cuda.Stream / raw handle -> cudaStream_t.  torch's default stream
    has handle 0, which the C ABI reads as "own stream": map it to
    cudaStreamLegacy (0x1) so work really runs on the caller's stream."""
    if stream is None:
        return None
    ptr = getattr(stream, "cuda_stream", stream)
    if hasattr(stream, "cuda_stream") and ptr == 0:
        return 1
    return ptr or None


def _dptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


# ---- model descriptions ------------------------------------------------------
def tree_data(tree) -> np.ndarray:
    """[M, root, (parent, left, right, age) x M] from a tree dict."""
    M = len(tree["age"])
    d = np.empty(2 + 4 * M, dtype=np.float64)
    d[0], d[1] = M, tree["root"]
    v = d[2:].reshape(M, 4)
    v[:, 0] = tree["parent"]
    v[:, 1] = tree["left"]
    v[:, 2] = tree["right"]
    v[:, 3] = tree["age"]
    return d


class Model:
    """Owns the host arrays an smc_model points at."""

    def __init__(self, kind, data=None, params=None, state_bytes=0, flags=0):
        self.kind = kind
        self.data = np.ascontiguousarray(data if data is not None else np.zeros(0), dtype=np.float64)
        self.params = np.ascontiguousarray(params if params is not None else np.zeros(0),
                                           dtype=np.float64)
        self.c = smc_model(kind, state_bytes, _dptr(self.data), self.data.size,
                           _dptr(self.params), self.params.size, flags)

    @staticmethod
    def crbd(tree, params=(1.0, -1.0, -1.0), flags=0, lineage=False, analytic=False):
        """analytic: the §5.3 variance reduction (2 E(t) per hidden event)."""
        return Model(CRBD, tree_data(tree), params,
                     flags=flags | (FLAG_LINEAGE_RNG if lineage else 0) | (FLAG_ANALYTIC_UNDETECTED if analytic else 0))

    @staticmethod
    def clads2(tree, params=(1.0, -1.0, -1.0, -1.0, -1.0), flags=0, lineage=False):  # noqa: D401
        return Model(CLADS2, tree_data(tree), params, flags=flags | (FLAG_LINEAGE_RNG if lineage else 0))

    @staticmethod
    def seir(y, params=None, flags=0):
        return Model(SEIR, np.asarray(y, dtype=np.float64), params, flags=flags)

    @staticmethod
    def ssm(y, params=(0.0, 100.0, 2.0, 1.0, 5.0), flags=0):
        return Model(SSM, np.asarray(y, dtype=np.float64), params, flags=flags)

    @staticmethod
    def geometric(p=0.5, w=1.5, flags=0):
        return Model(GEOMETRIC, None, (p, w), flags=flags)

    @staticmethod
    def fig3(p_loop=0.5, p3=0.3, w1=2.0, w2=1.2, w3=1.2, w4=0.5, flags=0):
        """The PCFG of Fig. 3(a) (R-23)."""
        return Model(FIG3, None, (p_loop, p3, w1, w2, w3, w4), flags=flags)

    @staticmethod
    def stackf(y, params=(2.0, 2.0, 0.5, 768.0), flags=0):
        """The recursive function of Fig. 5 compiled with a PSTATE byte stack
        (R-24): y = observation per recursion depth;
        params (p0, p_rec, sigma, stack bytes)."""
        return Model(STACKF, np.asarray(y, dtype=np.float64), params, flags=flags)

    @staticmethod
    def constw(logw=float(np.log(3.0)), K=1, flags=0):
        return Model(CONSTW, None, (logw, K), flags=flags)

    @staticmethod
    def resample_bench(state_bytes=64, flags=0):
        return Model(RESAMPLE_BENCH, None, None, state_bytes=state_bytes, flags=flags)


class Smc:
    """One SMC run over a PCFG model on the current CUDA device.

    shards > 1 emulates that many ranks on one GPU (the multi-GPU resampler
    path with virtual shards); n_particles is then the TOTAL count."""

    def __init__(self, model: Model, n_particles: int, seed: int = 1, shards: int = 1,
                 stream=None):
        self.model = model
        if shards == 1:
            self.h = _lib.smc_create(C.byref(model.c), int(n_particles), int(seed))
        else:
            if n_particles % shards:
                raise ValueError("n_particles must be divisible by shards")
            self.h = _lib.smc_create_virtual(C.byref(model.c), int(n_particles) // shards,
                                             int(seed), int(shards))
        if not self.h:
            raise SmcError(EINVAL, _lib.smc_errmsg(None).decode())
        self.n = int(n_particles)
        if stream is not None:
            self.set_stream(stream)

    def close(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.smc_destroy(self.h)
        self.h = None

    __del__ = close

    def set_stream(self, stream):
        """stream: torch.cuda.Stream, raw cudaStream_t int, or None."""
        _check(self.h, _lib.smc_set_stream(self.h, C.c_void_p(_stream_ptr(stream))))

    def set_data(self, data):
        d = np.ascontiguousarray(data, dtype=np.float64)
        self._data_keep = d
        _check(self.h, _lib.smc_set_data(self.h, _dptr(d), d.size))

    def set_ess_threshold(self, a, b):
        """Resample only when ESS < (a/b) N; a >= b: at every checkpoint."""
        _check(self.h, _lib.smc_set_ess_threshold(self.h, int(a), int(b)))

    def set_graph(self, on=True):
        _check(self.h, _lib.smc_set_graph(self.h, 1 if on else 0))

    def resample_grid(self):
        """CTAs of the single-launch fused resampling step (0: split kernels)."""
        v = C.c_int32(0)
        _check(self.h, _lib.smc_resample_grid(self.h, C.byref(v)))
        return v.value

    def set_timing(self, on=True):
        _check(self.h, _lib.smc_set_timing(self.h, 1 if on else 0))

    def reset(self, seed):
        _check(self.h, _lib.smc_reset(self.h, int(seed)))

    def run(self):
        return _check(self.h, _lib.smc_run(self.h))

    def run_status(self):
        """Run and return the status code instead of raising on EREJECTED/ENAN."""
        return _lib.smc_run(self.h)

    def step(self):
        done = C.c_int32(0)
        rc = _lib.smc_step(self.h, C.byref(done))
        return rc, bool(done.value)

    @property
    def log_z(self):
        return _lib.smc_log_z(self.h)

    def ancestors(self):
        out = np.empty(self.n, dtype=np.uint32)
        _check(self.h, _lib.smc_ancestors(self.h, out.ctypes.data_as(C.POINTER(C.c_uint32)), self.n))
        return out

    def log_weights(self):
        out = np.empty(self.n, dtype=np.float64)
        _check(self.h, _lib.smc_log_weights(self.h, _dptr(out), self.n))
        return out

    def fields(self):
        F = _lib.smc_nfields(self.h)
        out = np.empty((self.n, F), dtype=np.float64)
        _check(self.h, _lib.smc_fields(self.h, _dptr(out), out.size))
        return out

    def load(self, lw, state):
        """RESAMPLE_BENCH handles: numpy arrays (host) or torch CUDA tensors."""
        dev = hasattr(lw, "data_ptr")
        lp = lw.data_ptr() if dev else np.ascontiguousarray(lw, dtype=np.float64).ctypes.data
        if not dev:
            self._load_keep = (np.ascontiguousarray(lw, dtype=np.float64),
                               np.ascontiguousarray(state, dtype=np.uint8))
            lp, sp = self._load_keep[0].ctypes.data, self._load_keep[1].ctypes.data
        else:
            sp = state.data_ptr()
        _check(self.h, _lib.smc_load(self.h, C.c_void_p(lp), C.c_void_p(sp), 1 if dev else 0))

    def resample_step(self, epoch):
        _check(self.h, _lib.smc_resample_step(self.h, int(epoch)))

    def distinct(self):
        v = C.c_uint64(0)
        _check(self.h, _lib.smc_last_distinct(self.h, C.byref(v)))
        return v.value

    def state(self):
        st = self.stats()
        out = np.empty(st["state_bytes"] * self.n, dtype=np.uint8)
        _check(self.h, _lib.smc_state(self.h, out.ctypes.data, out.size))
        return out

    def stats(self):
        s = smc_stats_t()
        _check(self.h, _lib.smc_stats(self.h, C.byref(s)))
        d = {k: getattr(s, k) for k, _ in smc_stats_t._fields_}
        d["ms_kernel"] = list(d["ms_kernel"])
        return d


class Resampler:
    """Resampling step alone (BASELINE configs[4]) on n particles of
    state_bytes each.  State buffers are SoA planes: plane p of particle k at
    byte (p * n + k) * 16."""

    def __init__(self, n: int, state_bytes: int = 64, seed: int = 4, stream=None, inplace=False):
        """inplace: permuted ancestors, state updated in place (R-21);
        then device() takes state_out=None (or the same buffer as state_in)."""
        self.model = Model.resample_bench(state_bytes, FLAG_INPLACE if inplace else 0)
        self.h = _lib.smc_create(C.byref(self.model.c), int(n), int(seed))
        if not self.h:
            raise SmcError(EINVAL, _lib.smc_errmsg(None).decode())
        self.n, self.state_bytes = int(n), int(state_bytes)
        if stream is not None:
            _check(self.h, _lib.smc_set_stream(self.h, C.c_void_p(_stream_ptr(stream))))

    def close(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.smc_destroy(self.h)
        self.h = None

    __del__ = close

    def device(self, lw, state_in, state_out, anc, epoch=0, sync_logz=False):
        """Device pointers (ints) or torch tensors; enqueue only unless sync_logz."""
        ptr = [getattr(x, "data_ptr", lambda x=x: x)() for x in (lw, state_in, state_out, anc)]
        inc = C.c_double(0.0)
        _check(self.h, _lib.smc_resample_device(self.h, *[C.c_void_p(p) for p in ptr], int(epoch),
                                                C.byref(inc) if sync_logz else None))
        return inc.value if sync_logz else None

    def host(self, lw, states, epoch=0):
        """Host numpy arrays: lw float64[n], states uint8 SoA [planes, n, 16]."""
        lw = np.ascontiguousarray(lw, dtype=np.float64)
        states = np.ascontiguousarray(states, dtype=np.uint8)
        out = np.empty_like(states)
        anc = np.empty(self.n, dtype=np.uint32)
        inc = C.c_double(0.0)
        _check(self.h, _lib.smc_resample_host(self.h, _dptr(lw), states.ctypes.data, out.ctypes.data,
                                              anc.ctypes.data_as(C.POINTER(C.c_uint32)), int(epoch),
                                              C.byref(inc)))
        return anc, out, inc.value

    def set_timing(self, on=True):
        _check(self.h, _lib.smc_set_timing(self.h, 1 if on else 0))

    def stats(self):
        s = smc_stats_t()
        _check(self.h, _lib.smc_stats(self.h, C.byref(s)))
        d = {k: getattr(s, k) for k, _ in smc_stats_t._fields_}
        d["ms_kernel"] = list(d["ms_kernel"])
        return d

    def distinct(self):
        v = C.c_uint64(0)
        _check(self.h, _lib.smc_last_distinct(self.h, C.byref(v)))
        return v.value

    def resample_grid(self):
        """CTAs of the single-launch fused resampling step (0: split kernels)."""
        v = C.c_int32(0)
        _check(self.h, _lib.smc_resample_grid(self.h, C.byref(v)))
        return v.value


def plan_ranges(shard_totals, n_per: int, z: int):
    """Output slot range of each shard for integer shard totals (Python ints)
    and resampling integer z: returns out[0..world] (C++ planner, host only)."""
    world = len(shard_totals)
    w = np.zeros(2 * world, dtype=np.uint64)
    for g, W in enumerate(shard_totals):
        w[2 * g] = W & (2 ** 64 - 1)
        w[2 * g + 1] = W >> 64
    out = np.zeros(world + 1, dtype=np.uint64)
    _check(None, _lib.smc_plan_ranges(w.ctypes.data_as(C.POINTER(C.c_uint64)), world, int(n_per),
                                      int(z), out.ctypes.data_as(C.POINTER(C.c_uint64))))
    return [int(v) for v in out]


def draw_peak(draws_per_thread: int = 2048) -> float:
    """Measured draw-rate ceiling (uniforms/s) of the current device: the
    divergence-free Philox + hq + fp64 Exp microkernel (smc_draw_peak)."""
    v = C.c_double(0.0)
    _check(None, _lib.smc_draw_peak(int(draws_per_thread), C.byref(v)))
    return v.value


def aos_to_soa(states: np.ndarray) -> np.ndarray:
    """[n, S] bytes -> SoA planes [S/16, n, 16] (the library's layout)."""
    n, S = states.shape
    return np.ascontiguousarray(states.reshape(n, S // 16, 16).transpose(1, 0, 2))


def soa_to_aos(planes: np.ndarray) -> np.ndarray:
    P, n, _ = planes.shape
    return np.ascontiguousarray(planes.transpose(1, 0, 2).reshape(n, P * 16))
