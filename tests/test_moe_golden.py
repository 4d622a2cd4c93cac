"""CPU: the oracle's MoE arithmetic (oracle/moe_oracle.c, DESIGN.md Appendix A)
against fixtures generated from PUBLISHED GShard / Switch code (transformers
5.5.0 NllbMoeTop2Router.route_tokens, SwitchTransformersTop1Router,
load_balancing_loss_func, NllbMoeDenseActDense; tests/golden/make_moe_golden.py).
This is the independent pin of gating, capacity positions, drops, gates, aux
loss, expert FFN, combine and all of their gradients."""
import hashlib

import numpy as np
import pytest

import oracle
from moe_golden import LAYER, ROUTING, check_routing, load, routing_logits, tensor_errors


@pytest.mark.parametrize("name", sorted(ROUTING))
def test_oracle_routing_matches_published_routers(name):
    c = ROUTING[name]
    L = routing_logits(c["kind"], c["seed"], c["T"], c["E"], c["skew"])
    assert hashlib.sha256(L.tobytes()).hexdigest() == c["logits_sha256"], "input generator drifted"
    ref = load(name)
    got = oracle.route(L, c["k"], c["capacity"])
    check_routing(got, ref, gate_rtol=1e-12, aux_rtol=1e-6, tag=name)  # f_e is fp32 in load_balancing_loss_func


def test_c3_fixture_follows_gen_trace_skew():
    """c3's Gumbel-max logits give the top-1 histogram gen_trace's Zipf CDF
    would (workload.cpp:19-53): imbalance ratio within 3% of the reference's."""
    c = ROUTING["c3_route_zipf"]
    ref = load("c3_route_zipf")
    ir = ref["count1"].max() / ref["count1"].mean()
    tr = oracle.gen_trace(7, 1, 1, c["E"], c["T"], c["skew"])
    ir_ref = oracle.imbalance_ratio(tr)
    assert abs(ir / ir_ref - 1) < 0.03, (ir, ir_ref)
    assert (ref["keep"] == 0).sum() > 0


def _oracle_layer(c, ref):
    t = oracle.make_layer_tensors(c["seed"], c["T"], c["d"], c["dff"], c["E"], False,
                                  gate_bias=c["gate_bias"])
    fwd = oracle.moe_forward(t["x"], t["wg"], t["bg"], t["w1"], t["b1"], t["w2"], t["b2"],
                             c["k"], c["capacity"], False)
    if "logits" in ref:
        assert np.array_equal(fwd["logits"], ref["logits"])
    else:
        assert abs(fwd["logits"].astype(np.float64).sum() - ref["logits_sum"][0]) < 1e-6
    fwd["logits_used"] = fwd["logits"]
    bwd = oracle.moe_backward(t["x"], t["wg"], t["bg"], t["w1"], t["b1"], t["w2"], t["b2"],
                              c["k"], c["capacity"], False, fwd, t["dy"], c["d_aux"])
    return fwd, bwd


@pytest.mark.parametrize("name", [n for n in sorted(LAYER) if LAYER[n]["full"]])
def test_oracle_layer_matches_published_moe(name):
    c = LAYER[name]
    ref = load(name)
    fwd, bwd = _oracle_layer(c, ref)
    check_routing(fwd, ref, gate_rtol=1e-12, aux_rtol=1e-6, tag=name)
    got = dict(y=fwd["y"], **{n: bwd[n] for n in ("dx", "dwg", "dw1", "db1", "dw2", "db2",
                                                  "dbg")})
    errs = tensor_errors(got, ref)
    assert errs and all(v <= 1e-6 for v in errs.values()), errs


def test_oracle_layer_c1_full_size_matches_published_moe():
    """config c1 at full size (T=4096, E=8, top-2, d=512, d_ff=2048, cf=1.25)."""
    c = LAYER["layer_c1"]
    ref = load("layer_c1")
    fwd, bwd = _oracle_layer(c, ref)
    check_routing(fwd, ref, gate_rtol=1e-12, aux_rtol=1e-6, tag="layer_c1")
    got = dict(y=fwd["y"], **{n: bwd[n] for n in ("dx", "dwg", "dw1", "db1", "dw2", "db2")})
    errs = tensor_errors(got, ref)
    assert len(errs) == 14 and all(v <= 1e-6 for v in errs.values()), errs
