"""GPU: the CUDA gating / capacity / FFN / combine path and its backward against
fixtures from PUBLISHED GShard / Switch code (transformers 5.5.0 NLLB-MoE top-2
router, Switch top-1 router, load_balancing_loss_func, NLLB expert MLP;
tests/golden/make_moe_golden.py) — independent of the builder's oracle.

Routing integers bit-exact given identical fp32 logits; fp32 layer outputs and
gradients within 1e-5 * max|ref| per tensor (north_star)."""
import hashlib

import numpy as np
import pytest
import torch

from moe_golden import LAYER, ROUTING, check_routing, load, routing_logits, tensor_errors

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_2205_10034_b200 import MoEConfig, MoELayer, route  # noqa: E402
from paper_2205_10034_b200.layer import T_DY  # noqa: E402


@pytest.mark.parametrize("name", sorted(ROUTING))
def test_gpu_routing_matches_published_routers(name):
    c = ROUTING[name]
    L = routing_logits(c["kind"], c["seed"], c["T"], c["E"], c["skew"])
    assert hashlib.sha256(L.tobytes()).hexdigest() == c["logits_sha256"]
    got = route(torch.from_numpy(L).cuda(), c["k"], c["capacity"])
    torch.cuda.synchronize()
    got = {n: t.cpu().numpy() for n, t in got.items()}
    check_routing(got, load(name), tag=name)


@pytest.mark.parametrize("name", sorted(LAYER))
def test_gpu_fp32_layer_matches_published_moe(name):
    c = LAYER[name]
    ref = load(name)
    cfg = MoEConfig(c["E"], c["k"], c["d"], c["dff"], c["cf"], c["T"], torch.float32,
                    gate_bias=c["gate_bias"] is not None)
    layer = MoELayer(cfg)
    assert layer.capacity == c["capacity"]
    gb = None if c["gate_bias"] is None else torch.tensor(c["gate_bias"], dtype=torch.float32).cuda()
    layer.init_params(c["seed"], gate_bias=gb)
    x = layer.make_input(c["seed"])
    dy = layer.make_input(c["seed"], T_DY)
    y, rout = layer.forward(x, routing=True)
    dx = layer.backward(dy, d_aux=c["d_aux"])
    torch.cuda.synchronize()
    lg = rout["logits"].cpu().numpy().astype(np.float64)
    if "logits" in ref:
        assert np.abs(lg - ref["logits"]).max() <= 1e-5 * np.abs(ref["logits"]).max()
    else:
        assert abs(lg.sum() - ref["logits_sum"][0]) <= 1e-5 * np.abs(lg).sum()
    check_routing({n: t.cpu().numpy() for n, t in rout.items()}, ref, tag=name)
    g = layer.grads
    got = dict(y=y.cpu().numpy(), dx=dx.cpu().numpy(),
               **{n: g[n].cpu().numpy() for n in ("dwg", "dw1", "db1", "dw2", "db2")})
    if c["gate_bias"] is not None:
        got["dbg"] = g["dbg"].cpu().numpy()
    errs = tensor_errors(got, ref)
    assert errs and all(v <= 1e-5 for v in errs.values()), errs
