"""Gate-logit generators for the routing fixtures in tests/golden/moe/.

Used by make_moe_golden.py (to create the fixtures) and by the tests (to
regenerate the same fp32 logits on the GPU box, where neither transformers
nor /root/reference is needed).  Draws come from oracle.fill_uniform
(SplitMix64, rng.hpp:19-42); every kind except "gumbel_zipf" uses only exactly
rounded arithmetic, so the logits are bit-identical on any host.  The manifest
stores each case's sha256 so a host whose libm log differs is caught, not
silently mis-compared.
"""
from __future__ import annotations

import numpy as np

import oracle


def zipf_probs(E: int, skew: float) -> np.ndarray:
    """workload.cpp:19-53: p_e proportional to (e+1)^-skew."""
    w = np.array([(e + 1.0) ** -skew for e in range(E)])
    return w / w.sum()


def routing_logits(kind: str, seed: int, T: int, E: int, skew: float = 0.0) -> np.ndarray:
    n = T * E
    if kind == "uniform":
        L = oracle.fill_uniform(seed, n, -4.0, 4.0).astype(np.float64)
    elif kind in ("normal", "neg_inf"):
        u = oracle.fill_uniform(seed, 4 * n, 0.0, 1.0).astype(np.float64).reshape(4, n)
        L = (u.sum(0) - 2.0) * 1.7320508075688772  # Irwin-Hall(4), unit variance
        if kind == "neg_inf":
            m = oracle.fill_uniform(seed + 1, n, 0.0, 1.0).reshape(T, E) < 0.15
            m[:, :2] = False  # every row keeps >= 2 finite logits
            L = L.reshape(T, E)
            L[m] = -np.inf
    elif kind == "ties":
        L = np.floor(oracle.fill_uniform(seed, n, 0.0, 1.0).astype(np.float64) * 5.0) - 2.0
    elif kind == "gumbel_zipf":
        # Gumbel-max: argmax_e(ln p_e + G_te) ~ Categorical(p) — the same Zipf
        # top-1 distribution gen_trace draws token by token (workload.cpp:44-49).
        u = oracle.fill_uniform(seed, n, 0.0, 1.0).astype(np.float64)
        u = np.clip(u, 1e-12, 1.0 - 1e-12)
        g = -np.log(-np.log(u))
        L = g.reshape(T, E) + np.log(zipf_probs(E, skew))[None, :]
    else:
        raise ValueError(kind)
    return np.ascontiguousarray(np.asarray(L, np.float64).reshape(T, E).astype(np.float32))
