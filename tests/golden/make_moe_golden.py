"""Generate tests/golden/moe/*.npz from PUBLISHED GShard / Switch implementations.

The reference (moesim) has no MoE-layer arithmetic; the
paper names GShard / Switch routing.  transformers 5.5.0 in
this image carries both as published code, so this script pins the oracle's
Appendix A semantics (and, through the committed fixtures, the GPU kernels)
against them — independently of the builder's own restatement:

  * NllbMoeTop2Router.route_tokens
      (transformers/models/nllb_moe/modeling_nllb_moe.py:206-272)
      top-2 GShard router with second_expert_policy="all",
      normalize_router_prob_before_dropping=True, batch_prioritized_routing=False:
      locations1 = cumsum(top1)-1, locations2 = cumsum(top2)-1 + sum(top1),
      keep = location < expert_capacity, gates normalised over the two choices.
  * SwitchTransformersTop1Router.forward
      (transformers/models/switch_transformers/modeling_switch_transformers.py:80-107)
      top-1 router: argmax of the softmax, gate = max prob.  Its capacity mask is
      degenerate in 5.5 (see switch_route), so top-1 positions / drops come from
      the NLLB router's first-choice locations (the same GShard rule).
  * load_balancing_loss_func (modeling_switch_transformers.py:845-881), applied to
      the top-1 expert indices (GShard's l_aux uses the first choice only).
  * NllbMoeDenseActDense (modeling_nllb_moe.py:318-337): fc1 (+bias) -> act ->
      fc2 (+bias), with activation_function="gelu" (erf GeLU).
    transformers 5.5's NllbMoeExperts.forward one-hot-encodes the already
    one-hot top_1_mask (modeling_nllb_moe.py:350-360), so it is not used; the
    combine here is the NLLB/fairseq one: y_t = sum_e combine_weights[t,e] *
    expert_e(x_t) over the (token, expert) pairs the router kept.

Positions (slot index inside an expert's capacity buffer) are not returned by
either router; they are captured from the routers' own computations by
recording the arguments of the torch.lt calls NLLB's route_tokens makes
(locations1 / locations2 < expert_capacity).

Everything runs in float64 (router .dtype set to float64 after construction) on the fp32-rounded gate
logits, which is what the device stores and routes on ("bit-exact given
identical gate logits", north_star).  Backward = torch autograd of
loss = <y, dy> + d_aux * l_aux.

Inputs come from the SplitMix64 generators (rng.hpp:19-42) that the compiled
reference pins (tests/golden/reference_golden.json), via oracle.fill_uniform /
oracle.make_layer_tensors — so the GPU box can regenerate them without this
script or transformers.

    python tests/golden/make_moe_golden.py
"""
from __future__ import annotations

import hashlib
import json
import math
import os
import sys
from contextlib import contextmanager

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

import transformers  # noqa: E402
from transformers import NllbMoeConfig, SwitchTransformersConfig  # noqa: E402
from transformers.models.nllb_moe.modeling_nllb_moe import (  # noqa: E402
    NllbMoeDenseActDense, NllbMoeTop2Router)
from transformers.models.switch_transformers.modeling_switch_transformers import (  # noqa: E402
    SwitchTransformersTop1Router, load_balancing_loss_func)

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "moe")
torch.set_default_dtype(torch.float64)


# ------------------------------------------------------------------ inputs --
def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ----------------------------------------------------------------- routers --
@contextmanager
def record(fn_name):
    """Record every call of torch.<fn_name> made inside the block (the routers'
    own location / priority tensors)."""
    orig = getattr(torch, fn_name)
    calls = []

    def wrap(*a, **kw):
        out = orig(*a, **kw)
        calls.append((a, kw, out))
        return out

    setattr(torch, fn_name, wrap)
    try:
        yield calls
    finally:
        setattr(torch, fn_name, orig)


def nllb_route(logits: torch.Tensor, capacity: int):
    """Top-2: NllbMoeTop2Router.route_tokens on the given (float64) logits."""
    T, E = logits.shape
    cfg = NllbMoeConfig(d_model=E, num_experts=E, expert_capacity=capacity, router_bias=False,
                        router_dtype="float32", second_expert_policy="all",
                        normalize_router_prob_before_dropping=True,
                        batch_prioritized_routing=False, moe_eval_capacity_token_fraction=-1.0)
    r = NllbMoeTop2Router(cfg).eval()
    r.dtype = torch.float64  # config validation only admits 16/32-bit names; route in fp64
    with record("lt") as lt:
        top1_kept, combine = r.route_tokens(logits, torch.float64)
    loc1, loc2 = lt[0][0][0], lt[1][0][0]
    probs = torch.softmax(logits, dim=-1, dtype=torch.float64)
    # pre-drop choices: top-1 = argmax of the probabilities (route_tokens:219),
    # top-2 = argmax of the logits with the top-1 masked (route_tokens:226-228)
    e1 = torch.argmax(probs, dim=-1)
    e2 = torch.argmax(logits.masked_fill(torch.nn.functional.one_hot(e1, E).bool(),
                                         float("-inf")), dim=-1)
    expert = torch.stack([e1, e2], 1)
    pos = torch.stack([loc1.gather(1, e1[:, None])[:, 0], loc2.gather(1, e2[:, None])[:, 0]], 1)
    keep = pos < capacity
    assert torch.equal(top1_kept.gather(1, e1[:, None])[:, 0].bool(), keep[:, 0])
    # normalised gates before dropping; combine = gates * keep (route_tokens:264-268)
    pe = probs.gather(1, expert)
    gate = pe / torch.clamp(pe.sum(1, keepdim=True), min=torch.finfo(torch.float64).eps)
    cw = combine.gather(1, expert)
    assert torch.allclose(cw, gate * keep, rtol=0, atol=1e-15)
    return dict(expert=expert, position=pos, keep=keep, gate=gate, probs=probs, combine=combine)


def switch_route(logits: torch.Tensor, capacity: int):
    """Top-1: expert and gate from SwitchTransformersTop1Router.forward (identity
    classifier, so router_logits == the given logits); capacity position and
    keep from NllbMoeTop2Router's first-choice half (locations1 = cumsum(top1)-1,
    top_1_mask * (locations1 < capacity), modeling_nllb_moe.py:250-262).

    transformers 5.5's Switch router computes token_priority as a cumsum over a
    singleton axis (torch.max(..., keepdim=True) then one_hot adds an axis,
    modeling_switch_transformers.py:99-103), so its own capacity mask never
    drops a token; the GShard/Switch rule it intends is the NLLB one used here."""
    T, E = logits.shape
    cfg = SwitchTransformersConfig(d_model=E, num_experts=E, expert_capacity=capacity,
                                   router_bias=False, router_jitter_noise=0.0,
                                   router_dtype="float32")
    r = SwitchTransformersTop1Router(cfg).eval()
    r.dtype = torch.float64
    with torch.no_grad():
        r.classifier.weight.copy_(torch.eye(E))
    _, expert_index, max_prob = r(logits[None])
    e1 = expert_index.reshape(T, E).argmax(-1)  # the Switch router's choice (one-hot)
    top2 = nllb_route(logits, capacity) if E >= 2 else None
    probs = torch.softmax(logits, dim=-1, dtype=torch.float64)
    if top2 is None:  # E == 1: NLLB needs a second expert; one expert, positions = arange
        pos = torch.arange(T)[:, None]
    else:
        assert torch.equal(top2["expert"][:, 0], e1)
        pos = top2["position"][:, :1]
    keep = pos < capacity
    gate = max_prob.reshape(T, 1)
    return dict(expert=e1[:, None], position=pos, keep=keep, gate=gate, probs=probs,
                combine=None)


def route(logits: torch.Tensor, k: int, capacity: int):
    out = nllb_route(logits, capacity) if k == 2 else switch_route(logits, capacity)
    T, E = logits.shape
    e1 = out["expert"][:, 0]
    out["count1"] = torch.bincount(e1, minlength=E)
    out["count2"] = (torch.bincount(out["expert"][:, 1], minlength=E) if k == 2
                     else torch.zeros(E, dtype=torch.int64))
    out["kept"] = torch.clamp(out["count1"] + out["count2"], max=capacity)
    # load_balancing_loss_func(probs, top-1 indices) = E^2 * mean_e(f_e * P_e)
    out["aux_loss"] = load_balancing_loss_func(out["probs"][None], e1[None, :])
    return out


def routing_arrays(r, k):
    T = r["expert"].shape[0]
    return dict(expert=r["expert"].numpy().astype(np.int16),
                position=r["position"].numpy().astype(np.int32),
                keep=r["keep"].numpy().astype(np.uint8),
                gate=r["gate"].detach().numpy().astype(np.float64).reshape(T, k),
                count1=r["count1"].numpy().astype(np.int32),
                count2=r["count2"].numpy().astype(np.int32),
                kept=r["kept"].numpy().astype(np.int32),
                aux_loss=np.float64(r["aux_loss"].item()))


# ------------------------------------------------------------------ layer --
def nllb_expert(d, dff, w1, b1, w2, b2):
    cfg = NllbMoeConfig(d_model=d, activation_function="gelu", activation_dropout=0.0)
    m = NllbMoeDenseActDense(cfg, dff).eval()
    m.fc1.weight = torch.nn.Parameter(torch.from_numpy(w1.astype(np.float64)))
    m.fc1.bias = torch.nn.Parameter(torch.from_numpy(b1.astype(np.float64)))
    m.fc2.weight = torch.nn.Parameter(torch.from_numpy(w2.astype(np.float64)))
    m.fc2.bias = torch.nn.Parameter(torch.from_numpy(b2.astype(np.float64)))
    return m


def layer_case(seed, T, d, dff, E, k, cf, d_aux, gate_bias=None):
    t = oracle.make_layer_tensors(seed, T, d, dff, E, False, gate_bias=gate_bias)
    cap = int(math.ceil(k * cf * T / E))
    x = torch.from_numpy(t["x"].astype(np.float64)).requires_grad_(True)
    dy = torch.from_numpy(t["dy"].astype(np.float64))
    # gate projection = the NLLB router classifier (nn.Linear, router_bias)
    cls = torch.nn.Linear(d, E, bias=gate_bias is not None)
    cls.weight = torch.nn.Parameter(torch.from_numpy(t["wg"].astype(np.float64)))
    if gate_bias is not None:
        cls.bias = torch.nn.Parameter(torch.from_numpy(t["bg"].astype(np.float64)))
    l64 = cls(x)
    l32 = l64.detach().float().double()
    logits = l64 + (l32 - l64).detach()  # routes on the fp32-rounded logits, grads flow
    r = route(logits, k, cap)
    experts = [nllb_expert(d, dff, t["w1"][e], t["b1"][e], t["w2"][e], t["b2"][e])
               for e in range(E)]
    y = torch.zeros(T, d)
    for e in range(E):
        for i in range(k):
            sel = ((r["expert"][:, i] == e) & r["keep"][:, i]).nonzero()[:, 0]
            if len(sel):
                y = y.index_add(0, sel, r["gate"][sel, i:i + 1] * experts[e](x[sel]))
    loss = (y * dy).sum() + d_aux * r["aux_loss"]
    loss.backward()
    def grad(p):  # an expert that received no token has no autograd grad
        return torch.zeros_like(p) if p.grad is None else p.grad

    g = dict(dx=x.grad, dwg=cls.weight.grad,
             dw1=torch.stack([grad(m.fc1.weight) for m in experts]),
             db1=torch.stack([grad(m.fc1.bias) for m in experts]),
             dw2=torch.stack([grad(m.fc2.weight) for m in experts]),
             db2=torch.stack([grad(m.fc2.bias) for m in experts]))
    if gate_bias is not None:
        g["dbg"] = cls.bias.grad
    out = routing_arrays(r, k)
    out["logits"] = l32.numpy().astype(np.float32)
    out["y"] = y.detach().numpy()
    for n, v in g.items():
        out[n] = v.detach().numpy()
    return out, cap


def summarise(out, full: bool, row_stride: dict):
    """Full float tensors for small cases; for big ones, every s-th row along
    axis -2 (fp32) plus float64 whole-tensor sum / abs-sum / max-abs."""
    res = {}
    for n, v in out.items():
        if n in ("y", "dx", "dwg", "dw1", "db1", "dw2", "db2", "dbg"):
            v = np.asarray(v, np.float64)
            res[n + "_sum"] = np.array([v.sum(), np.abs(v).sum(), np.abs(v).max()])
            if full or n not in row_stride:
                res[n] = v.astype(np.float32)
            else:
                s = row_stride[n]
                res[n + "_rows"] = v[..., ::s, :].astype(np.float32)
                res[n + "_stride"] = np.int32(s)
        else:
            res[n] = v
    return res


def main():
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from moe_inputs import routing_logits as gen_logits  # noqa: E402
    os.makedirs(OUT, exist_ok=True)
    manifest = {"transformers": transformers.__version__, "torch": torch.__version__,
                "routing": [], "layer": []}

    # ---- routing-only cases (logits regenerated by the tests) -------------
    rcases = [
        ("c1_route", "uniform", 11, 4096, 8, 2, 1.25, 0.0),      # config c1 shape
        ("c2_route", "uniform", 12, 65536, 64, 1, 1.25, 0.0),    # config c2 shape
        ("c3_route_zipf", "gumbel_zipf", 13, 65536, 32, 2, 1.25, 1.2),  # config c3: gen_trace skew
        ("ragged_top2", "normal", 14, 1000, 64, 2, 1.0, 0.0),
        ("e2_heavy_drops", "normal", 15, 257, 2, 2, 0.5, 0.0),
        ("e256_top1", "normal", 16, 3000, 256, 1, 2.0, 0.0),
        ("single_token", "normal", 17, 1, 4, 1, 1.0, 0.0),
        ("ties_top1", "ties", 18, 2048, 16, 1, 1.17, 0.0),
        ("ties_top2", "ties", 18, 2048, 16, 2, 1.17, 0.0),
        ("neg_inf_top2", "neg_inf", 19, 2048, 16, 2, 1.25, 0.0),
        ("zero_capacity", "normal", 20, 600, 8, 2, 0.0, 0.0),
    ]
    for name, kind, seed, T, E, k, cf, skew in rcases:
        L = gen_logits(kind, seed, T, E, skew)
        cap = int(math.ceil(k * cf * T / E))
        r = route(torch.from_numpy(L.astype(np.float64)), k, cap)
        arr = routing_arrays(r, k)
        np.savez_compressed(os.path.join(OUT, name + ".npz"), **arr)
        manifest["routing"].append(dict(name=name, kind=kind, seed=seed, T=T, E=E, k=k, cf=cf,
                                        skew=skew, capacity=cap, logits_sha256=sha(L),
                                        dropped=int((arr["keep"] == 0).sum())))
        print(name, "cap", cap, "dropped", int((arr["keep"] == 0).sum()), flush=True)

    # ---- layer cases (inputs from oracle.make_layer_tensors) ---------------
    lcases = [
        ("layer_top2_small", 1234, 256, 64, 128, 8, 2, 1.25, 0.05, None, True),
        ("layer_top1_drops", 1235, 512, 64, 128, 16, 1, 0.75, 0.05, None, True),
        ("layer_top2_bias_skew", 1236, 384, 64, 128, 32, 2, 1.25, 0.02,
         [-1.2 * math.log(e + 1.0) for e in range(32)], True),
        ("layer_c1", 2205, 4096, 512, 2048, 8, 2, 1.25, 0.05, None, False),
    ]
    for name, seed, T, d, dff, E, k, cf, d_aux, bias, full in lcases:
        out, cap = layer_case(seed, T, d, dff, E, k, cf, d_aux, bias)
        res = summarise(out, full, {"y": 32, "dx": 32, "dw1": 64, "dw2": 64})
        if not full:
            res.pop("logits")  # regenerated: GPU / oracle logits are checked against l_sum
            res["logits_sum"] = np.array([out["logits"].astype(np.float64).sum()])
        np.savez_compressed(os.path.join(OUT, name + ".npz"), **res)
        manifest["layer"].append(dict(name=name, seed=seed, T=T, d=d, dff=dff, E=E, k=k, cf=cf,
                                      d_aux=d_aux, gate_bias=bias, capacity=cap, full=full,
                                      dropped=int((out["keep"] == 0).sum())))
        print(name, "cap", cap, "dropped", int((out["keep"] == 0).sum()), "count1",
              out["count1"].tolist(), flush=True)

    with open(os.path.join(OUT, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1)


if __name__ == "__main__":
    main()
