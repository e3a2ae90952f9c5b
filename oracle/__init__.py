"""ctypes binding of the sequential CPU oracle (``oracle/smc_oracle.cpp``).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with ``paper_2112_00364_b200`` (the CUDA path) and
neither imports the other.

Every function here is argument marshalling; the arithmetic is in the C++ file,
each part of which cites the PAPER.md passage it follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "smc_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

# model kinds (same numbering as the public header, redeclared here on purpose)
CRBD, CLADS2, SEIR, CRBD_LR, CLADS2_LR, CRBD_AE, GEOMETRIC, SSM, CONSTW, FIG3, STACKF = (
    1, 2, 3, 4, 5, 6, 10, 11, 12, 13, 14)
OK, EINVAL, EREJECTED, ENAN = 0, 1, 4, 5
DIST = {"exp": 0, "bernoulli": 1, "uniform": 2, "normal": 3, "gamma": 4, "beta": 5, "binomial": 6}


def build(force: bool = False) -> str:
    """Compile the oracle with -O2 -ffp-contract=off (no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fPIC", "-shared",
               "-o", _LIB + ".tmp", _SRC]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_LIB)
            P = C.POINTER
            d, u32, u64, i32, i64, vp = C.c_double, C.c_uint32, C.c_uint64, C.c_int, C.c_int64, C.c_void_p
            L.oracle_errmsg.restype = C.c_char_p
            L.oracle_philox.argtypes = [P(u32), P(u32), P(u32)]
            L.oracle_uniforms.argtypes = [u64, u32, u32, u32, u64, P(d)]
            L.oracle_sample.argtypes = [i32, P(d), u64, u64, P(d), P(u32)]
            L.oracle_binomial_logpmf.argtypes = [i64, i64, d]
            L.oracle_binomial_logpmf.restype = d
            L.oracle_crbd_E.argtypes = [d, d, d, d]
            L.oracle_crbd_E.restype = d
            L.oracle_normal_logpdf.argtypes = [d, d, d]
            L.oracle_normal_logpdf.restype = d
            L.oracle_u128_to_double.argtypes = [u64, u64]
            L.oracle_u128_to_double.restype = d
            L.oracle_resample.argtypes = [P(d), u64, u64, u32, P(u32), P(u64), P(d), P(d), P(u64)]
            L.oracle_systematic.argtypes = [P(u64), u64, u64, P(u32)]
            L.oracle_quantize.argtypes = [P(d), u64, P(u64)]
            L.oracle_gather.argtypes = [vp, vp, P(u32), u64, u64]
            L.oracle_permute.argtypes = [P(u32), u64, P(u32)]
            L.oracle_smc_set_inplace.argtypes = [vp, i32]
            L.oracle_smc_create.argtypes = [i32, P(d), u64, P(d), i32, u64, u64]
            L.oracle_smc_create.restype = vp
            L.oracle_smc_step.argtypes = [vp, P(i32)]
            L.oracle_smc_run.argtypes = [vp]
            L.oracle_smc_set_ess.argtypes = [vp, u32, u32]
            L.oracle_smc_last_ess.argtypes = [vp]
            L.oracle_smc_last_ess.restype = d
            L.oracle_ess_gate.argtypes = [P(d), u64, u32, u32, P(d)]
            L.oracle_smc_log_z.argtypes = [vp]
            L.oracle_smc_log_z.restype = d
            L.oracle_smc_epoch.argtypes = [vp]
            L.oracle_smc_epoch.restype = u32
            L.oracle_smc_nfields.argtypes = [vp]
            L.oracle_smc_fields.argtypes = [vp, P(d)]
            L.oracle_smc_lw.argtypes = [vp, P(d)]
            L.oracle_smc_anc.argtypes = [vp, P(u32)]
            L.oracle_smc_stats.argtypes = [vp, P(u64)]
            L.oracle_smc_destroy.argtypes = [vp]
            L.oracle_gen_yule.argtypes = [u64, i32, d, d, P(i32), P(i32), P(i32), P(d)]
            L.oracle_gen_yule.restype = i64
            L.oracle_gen_seir.argtypes = [u64, i32, P(d), P(i64), P(i64)]
            L.oracle_gen_seir.restype = i64
            L.oracle_gen_ssm.argtypes = [u64, i32, P(d), P(d), P(d)]
            L.oracle_gen_ssm.restype = i64
            _lib = L
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


class OracleError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"oracle status {code} {msg}")
        self.code = code


# ---------------------------------------------------------------------------
def philox(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().oracle_philox(_p(c, C.c_uint32), _p(k, C.c_uint32), _p(out, C.c_uint32))
    return out


def uniforms(seed, particle, epoch, tag, n):
    out = np.zeros(n, dtype=np.float64)
    lib().oracle_uniforms(seed, particle, epoch, tag, n, _p(out, C.c_double))
    return out


def sample(dist, params, seed, n):
    """n variates; variate i uses particle stream i.  Returns (values, draws)."""
    prm = np.asarray(params, dtype=np.float64)
    out = np.zeros(n, dtype=np.float64)
    dr = np.zeros(n, dtype=np.uint32)
    rc = lib().oracle_sample(DIST[dist], _p(prm, C.c_double), seed, n, _p(out, C.c_double),
                             _p(dr, C.c_uint32))
    if rc:
        raise OracleError(rc)
    return out, dr


def binomial_logpmf(k, n, p):
    return lib().oracle_binomial_logpmf(int(k), int(n), float(p))


def normal_logpdf(y, mu, s):
    return lib().oracle_normal_logpdf(float(y), float(mu), float(s))


def u128_to_double(x: int) -> float:
    return lib().oracle_u128_to_double(x & (2**64 - 1), x >> 64)


def resample(lw, seed, epoch):
    """Exact systematic resampling of log-weights lw (reading R1).

    Returns dict(anc, W, m, logz_inc, z)."""
    lw = np.ascontiguousarray(lw, dtype=np.float64)
    N = lw.size
    anc = np.zeros(N, dtype=np.uint32)
    W = np.zeros(2, dtype=np.uint64)
    m = C.c_double()
    inc = C.c_double()
    z = C.c_uint64()
    rc = lib().oracle_resample(_p(lw, C.c_double), N, seed, epoch, _p(anc, C.c_uint32),
                               _p(W, C.c_uint64), C.byref(m), C.byref(inc), C.byref(z))
    if rc:
        raise OracleError(rc)
    return dict(anc=anc, W=int(W[0]) | (int(W[1]) << 64), m=m.value, logz_inc=inc.value,
                z=z.value)


def systematic(q, z):
    """Ancestors for integer weights q (uint64) and resample integer z."""
    q = np.ascontiguousarray(q, dtype=np.uint64)
    anc = np.zeros(q.size, dtype=np.uint32)
    rc = lib().oracle_systematic(_p(q, C.c_uint64), q.size, int(z), _p(anc, C.c_uint32))
    if rc:
        raise OracleError(rc)
    return anc


def ess_gate(lw, a, b):
    """(resample?, ESS) for log-weights lw and threshold a/b (exact gate)."""
    lw = np.ascontiguousarray(lw, dtype=np.float64)
    e = C.c_double()
    rc = lib().oracle_ess_gate(_p(lw, C.c_double), lw.size, a, b, C.byref(e))
    if rc < 0:
        raise OracleError(-rc)
    return bool(rc), e.value


def quantize(lw):
    lw = np.ascontiguousarray(lw, dtype=np.float64)
    q = np.zeros(lw.size, dtype=np.uint64)
    rc = lib().oracle_quantize(_p(lw, C.c_double), lw.size, _p(q, C.c_uint64))
    if rc:
        raise OracleError(rc)
    return q


def gather(states, anc):
    """states: uint8 [N, S]; returns states[anc] computed by the oracle."""
    states = np.ascontiguousarray(states, dtype=np.uint8)
    anc = np.ascontiguousarray(anc, dtype=np.uint32)
    out = np.zeros_like(states)
    lib().oracle_gather(states.ctypes.data, out.ctypes.data, _p(anc, C.c_uint32), anc.size,
                        states.shape[1])
    return out


def permute(anc_sorted):
    """In-place ancestor permutation (R-21) of sorted ancestors."""
    a = np.ascontiguousarray(anc_sorted, dtype=np.uint32)
    c = np.zeros_like(a)
    lib().oracle_permute(_p(a, C.c_uint32), a.size, _p(c, C.c_uint32))
    return c


def tree_blob(tree) -> np.ndarray:
    """Oracle-side encoding of a tree dict (parent/left/right/age/root)."""
    M = len(tree["age"])
    d = [float(M), float(tree["root"])]
    for i in range(M):
        d += [float(tree["parent"][i]), float(tree["left"][i]), float(tree["right"][i]),
              float(tree["age"][i])]
    return np.asarray(d, dtype=np.float64)


class Smc:
    """Sequential SMC run of one model (Alg. 1 with the RootPPL loop order)."""

    def __init__(self, kind, data, params, n_particles, seed):
        data = np.ascontiguousarray(data if data is not None else np.zeros(0), dtype=np.float64)
        prm = np.ascontiguousarray(params if params is not None else np.zeros(0), dtype=np.float64)
        self._keep = (data, prm)
        self.N = int(n_particles)
        self.h = lib().oracle_smc_create(kind, _p(data, C.c_double), data.size,
                                         _p(prm, C.c_double), prm.size, self.N, seed)
        if not self.h:
            raise OracleError(EINVAL, lib().oracle_errmsg().decode())

    def __del__(self):
        if getattr(self, "h", None):
            lib().oracle_smc_destroy(self.h)
            self.h = None

    def step(self):
        done = C.c_int(0)
        rc = lib().oracle_smc_step(self.h, C.byref(done))
        return rc, bool(done.value)

    def run(self):
        return lib().oracle_smc_run(self.h)

    def set_inplace(self, on=True):
        """Permuted ancestors for in-place resampling (R-21)."""
        lib().oracle_smc_set_inplace(self.h, 1 if on else 0)

    def set_ess(self, a, b):
        """ESS threshold tau = a / b (a >= b: resample at every checkpoint)."""
        rc = lib().oracle_smc_set_ess(self.h, a, b)
        if rc:
            raise OracleError(rc)

    @property
    def last_ess(self):
        return lib().oracle_smc_last_ess(self.h)

    @property
    def log_z(self):
        return lib().oracle_smc_log_z(self.h)

    @property
    def epoch(self):
        return lib().oracle_smc_epoch(self.h)

    def lw(self):
        out = np.zeros(self.N, dtype=np.float64)
        lib().oracle_smc_lw(self.h, _p(out, C.c_double))
        return out

    def anc(self):
        out = np.zeros(self.N, dtype=np.uint32)
        lib().oracle_smc_anc(self.h, _p(out, C.c_uint32))
        return out

    def fields(self):
        F = lib().oracle_smc_nfields(self.h)
        out = np.zeros((self.N, F), dtype=np.float64)
        lib().oracle_smc_fields(self.h, _p(out, C.c_double))
        return out

    def stats(self):
        out = np.zeros(7, dtype=np.uint64)
        lib().oracle_smc_stats(self.h, _p(out, C.c_uint64))
        keys = ["epochs", "resamples", "draws", "overflow", "alive_particle_steps", "status",
                "guard"]
        return {k: int(v) for k, v in zip(keys, out)}


def gen_yule(seed, ntips, lam0=1.0, crown_age=30.0):
    M = 2 * ntips - 1
    par = np.zeros(M, dtype=np.int32)
    lef = np.zeros(M, dtype=np.int32)
    rig = np.zeros(M, dtype=np.int32)
    age = np.zeros(M, dtype=np.float64)
    used = lib().oracle_gen_yule(seed, ntips, lam0, crown_age, _p(par, C.c_int), _p(lef, C.c_int),
                                 _p(rig, C.c_int), _p(age, C.c_double))
    return dict(parent=par.tolist(), left=lef.tolist(), right=rig.tolist(), age=age.tolist(),
                root=0), int(used)


def gen_seir(seed, T, params):
    prm = np.asarray(params, dtype=np.float64)
    y = np.zeros(T, dtype=np.int64)
    z = np.zeros(T, dtype=np.int64)
    used = lib().oracle_gen_seir(seed, T, _p(prm, C.c_double), _p(y, C.c_int64), _p(z, C.c_int64))
    return y, z, int(used)


def gen_ssm(seed, T, params=(0.0, 100.0, 2.0, 1.0, 5.0)):
    prm = np.asarray(params, dtype=np.float64)
    y = np.zeros(T, dtype=np.float64)
    x = np.zeros(T, dtype=np.float64)
    used = lib().oracle_gen_ssm(seed, T, _p(prm, C.c_double), _p(y, C.c_double), _p(x, C.c_double))
    return y, x, int(used)
