"""Shared loader for the published-implementation fixtures in tests/golden/moe/
(made by tests/golden/make_moe_golden.py from transformers' NLLB-MoE / Switch
routers, load-balancing loss and NLLB expert MLP; see that script's header).

Tolerances (north_star):
  integers (expert, position, keep, counts): bit-exact
  fp32 paths: max|got - ref| <= 1e-5 * max|ref| per tensor
  gates: rtol 2e-6 (fp32 exp/div on the device), aux loss rtol 1e-5
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "moe")
sys.path.insert(0, os.path.join(HERE, "golden"))
from moe_inputs import routing_logits  # noqa: E402,F401

with open(os.path.join(GOLD, "manifest.json")) as f:
    MANIFEST = json.load(f)
ROUTING = {c["name"]: c for c in MANIFEST["routing"]}
LAYER = {c["name"]: c for c in MANIFEST["layer"]}
INT_KEYS = ("expert", "position", "keep", "count1", "count2", "kept")
GRAD_KEYS = ("dx", "dwg", "dw1", "db1", "dw2", "db2", "dbg")


def load(name):
    z = np.load(os.path.join(GOLD, name + ".npz"))
    return {k: z[k] for k in z.files}


def check_routing(got, ref, gate_rtol=2e-6, aux_rtol=1e-5, tag=""):
    for n in INT_KEYS:
        a = np.asarray(got[n]).astype(np.int64).reshape(ref[n].shape)
        assert np.array_equal(a, ref[n].astype(np.int64)), f"{tag}: {n} differs"
    np.testing.assert_allclose(np.asarray(got["gate"], np.float64).reshape(ref["gate"].shape),
                               ref["gate"], rtol=gate_rtol, atol=gate_rtol * 1e-1,
                               err_msg=f"{tag}: gate")
    np.testing.assert_allclose(float(np.asarray(got["aux_loss"]).reshape(-1)[0]),
                               float(ref["aux_loss"]), rtol=aux_rtol, err_msg=f"{tag}: aux")


def tensor_errors(got: dict, ref: dict) -> dict:
    """Per-tensor relative error vs the fixture: full tensors when stored, else
    the stored rows (normalised by the whole tensor's max|ref|) and the
    whole-tensor sum (normalised by sum|ref|)."""
    errs = {}
    for n in ("y",) + GRAD_KEYS:
        if n + "_sum" not in ref or n not in got:
            continue
        g = np.asarray(got[n], np.float64)
        s = ref[n + "_sum"]
        if n in ref:
            errs[n] = float(np.abs(g - ref[n]).max() / max(s[2], 1e-30))
        else:
            st = int(ref[n + "_stride"])
            rows = g[..., ::st, :]
            errs[n] = float(np.abs(rows - ref[n + "_rows"]).max() / max(s[2], 1e-30))
        errs[n + "_sum"] = float(abs(g.sum() - s[0]) / max(s[1], 1e-30))
    return errs
