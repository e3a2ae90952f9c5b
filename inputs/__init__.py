"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic: it only loads the committed
fixture files (trees, case series, observation series — written once by
``oracle/gen_inputs.py``) and draws synthetic log-weights / state bytes for the
resampling microbenchmark (BASELINE.json configs[4]) from numpy's PCG64.
Neither ``oracle`` nor ``paper_2112_00364_b200`` is imported here.
"""
from __future__ import annotations

import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def _load(name):
    with open(os.path.join(HERE, name)) as f:
        return json.load(f)


def tree(name: str = "tree90") -> dict:
    """Tree dict: root, parent[], left[], right[], age[] (tips: left = right = -1)."""
    return _load(f"{name}.json")


def seir_series(name: str = "seir182") -> np.ndarray:
    return np.asarray(_load(f"{name}.json")["y"], dtype=np.float64)


def ssm_series(T: int = 10) -> np.ndarray:
    return np.asarray(_load(f"ssm{T}.json")["y"], dtype=np.float64)


def stackf_series(name: str = "stackf12") -> np.ndarray:
    return np.asarray(_load(f"{name}.json")["y"], dtype=np.float64)


def resample_lw(n: int, sigma: float = 1.0, frac_neg_inf: float = 0.0, seed: int = 4) -> np.ndarray:
    """C4 log-weights: lw_k = sigma * N(0,1); a fraction set to -inf."""
    g = np.random.Generator(np.random.PCG64(seed))
    lw = sigma * g.standard_normal(n)
    if frac_neg_inf > 0:
        lw[g.random(n) < frac_neg_inf] = -np.inf
    return lw


def state_bytes(n: int, s: int = 64, seed: int = 5) -> np.ndarray:
    """C4 particle states: n x s random bytes."""
    g = np.random.Generator(np.random.PCG64(seed))
    return g.integers(0, 256, size=(n, s), dtype=np.uint8)


# Model parameter vectors used by tests and the bench (one definition, both
# sides read it; these are inputs, not arithmetic).
CRBD_PARAMS = [1.0, -1.0, -1.0]                 # rho, lambda_fixed (<0: prior), mu_fixed
CLADS2_PARAMS = [1.0, -1.0, -1.0, -1.0, -1.0]   # rho, lambda0, sigma, alpha, eps (<0: prior)
SSM_PARAMS = [0.0, 100.0, 2.0, 1.0, 5.0]        # m0, s0, drift, q, r (std devs)
GEOMETRIC_PARAMS = [0.5, 1.5]                   # p, w  (Fig. 2)
CONSTW_PARAMS = [float(np.log(3.0)), 4.0]       # log w, K checkpoints
FIG3_PARAMS = [0.5, 0.3, 2.0, 1.2, 1.2, 0.5]    # p_loop, p3, w1, w2, w3, w4 (Fig. 3(a) PCFG)
STACKF_PARAMS = [2.0, 2.0, 0.5, 768.0]          # p0, p_rec, sigma, stack bytes (Fig. 5(c) program)
