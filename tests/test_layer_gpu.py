"""GPU: the full MoE layer (forward + backward) through the C-ABI against the
fp64 CPU oracle (DESIGN.md Appendix A) on identical SplitMix64-generated
inputs.  Routing integers must be bit-exact given the GPU's fp32 logits;
float outputs and gradients within the north-star tolerances:
    fp32: max|got - ref| <= 1e-5 * max|ref|    (per tensor)
    bf16: max|got - ref| <= 2e-2 * max|ref|    (oracle emulates the bf16 stores)
At full config size the oracle is too slow; there a torch fp32 reference of
the same layer, built on the GPU's own routing, checks the numerics."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_2205_10034_b200 import MoEConfig, MoELayer  # noqa: E402
from paper_2205_10034_b200.layer import T_DY  # noqa: E402

TOL = {torch.float32: 1e-5, torch.bfloat16: 2e-2}


def rel_err(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30))


def run_case(E, k, d, dff, T, cf, dtype, seed=1234, d_aux=0.05, gate_bias=None):
    cfg = MoEConfig(E, k, d, dff, cf, T, dtype, gate_bias=gate_bias is not None)
    layer = MoELayer(cfg)
    gb = None if gate_bias is None else torch.tensor(gate_bias, dtype=torch.float32).cuda()
    layer.init_params(seed, gate_bias=gb)
    x = layer.make_input(seed)
    dy = layer.make_input(seed, T_DY)
    y, rout = layer.forward(x, routing=True)
    dx = layer.backward(dy, d_aux=d_aux)
    torch.cuda.synchronize()
    bf16 = dtype == torch.bfloat16
    ref_t = oracle.make_layer_tensors(seed, T, d, dff, E, bf16, gate_bias=gate_bias)
    # inputs are bit-identical
    assert np.array_equal(x.float().cpu().numpy(), ref_t["x"])
    assert np.array_equal(layer.params["w1"].float().cpu().numpy(), ref_t["w1"])
    g_logits = rout["logits"].cpu().numpy()
    fwd = oracle.moe_forward(ref_t["x"], ref_t["wg"], ref_t["bg"], ref_t["w1"], ref_t["b1"],
                             ref_t["w2"], ref_t["b2"], k, layer.capacity, bf16,
                             logits_in=g_logits)
    fwd["logits_used"] = g_logits
    return layer, x, y, dx, rout, fwd, ref_t, d_aux


def check_case(E, k, d, dff, T, cf, dtype, **kw):
    layer, x, y, dx, rout, fwd, ref_t, d_aux = run_case(E, k, d, dff, T, cf, dtype, **kw)
    tol = TOL[dtype]
    # K1: logits vs fp64-accumulated logits
    assert rel_err(rout["logits"].cpu().numpy(), fwd["logits"]) < (1e-5 if dtype == torch.float32 else 1e-4)
    # K2: routing bit-exact given the GPU logits
    for n in ("expert", "position", "count1", "count2", "kept", "keep"):
        assert np.array_equal(rout[n].cpu().numpy(), fwd[n]), n
    np.testing.assert_allclose(rout["gate"].cpu().numpy(), fwd["gate"], rtol=2e-6, atol=1e-7)
    np.testing.assert_allclose(rout["aux_loss"].item(), fwd["aux_loss"], rtol=1e-5)
    # forward output
    assert rel_err(y.float().cpu().numpy(), fwd["y"]) <= tol
    # backward
    bwd = oracle.moe_backward(ref_t["x"], ref_t["wg"], ref_t["bg"], ref_t["w1"], ref_t["b1"],
                              ref_t["w2"], ref_t["b2"], k, layer.capacity, dtype == torch.bfloat16,
                              fwd, ref_t["dy"], d_aux)
    g = layer.grads
    checks = {
        "dx": (dx.float().cpu().numpy(), bwd["dx"]),
        "dwg": (g["dwg"].cpu().numpy(), bwd["dwg"]),
        "dw1": (g["dw1"].cpu().numpy(), bwd["dw1"]),
        "db1": (g["db1"].cpu().numpy(), bwd["db1"]),
        "dw2": (g["dw2"].cpu().numpy(), bwd["dw2"]),
        "db2": (g["db2"].cpu().numpy(), bwd["db2"]),
    }
    if kw.get("gate_bias") is not None:
        checks["dbg"] = (g["dbg"].cpu().numpy(), bwd["dbg"])
    errs = {n: rel_err(a, b) for n, (a, b) in checks.items()}
    bad = {n: e for n, e in errs.items() if not e <= tol}
    assert not bad, errs
    return layer, fwd


def test_layer_bf16_top2_small():
    check_case(E=8, k=2, d=256, dff=512, T=512, cf=1.25, dtype=torch.bfloat16)


def test_layer_bf16_top1_switch_shape():
    # config c2 ratios (E=64, top-1, d_ff = 4 d) at reduced size
    check_case(E=64, k=1, d=128, dff=512, T=2048, cf=1.25, dtype=torch.bfloat16)


def test_layer_bf16_skewed_drops_c3():
    E = 32
    bias = [-1.2 * np.log(e + 1.0) for e in range(E)]
    layer, fwd = check_case(E=E, k=2, d=128, dff=256, T=1024, cf=1.25, dtype=torch.bfloat16,
                            gate_bias=bias)
    assert (fwd["keep"] == 0).sum() > 0  # capacity drops exercised


def test_layer_fp32_c1_shape():
    # config c1 (E=8 top-2 d=512 d_ff=2048 cf=1.25, fp32) at T=512 (oracle cost)
    check_case(E=8, k=2, d=512, dff=2048, T=512, cf=1.25, dtype=torch.float32)


def test_layer_fp32_drops():
    check_case(E=4, k=2, d=64, dff=128, T=300, cf=0.5, dtype=torch.float32)


def test_layer_ragged_tokens_bf16():
    # T not a multiple of the routing chunk / GEMM tile, tiny experts
    check_case(E=16, k=2, d=128, dff=256, T=333, cf=2.0, dtype=torch.bfloat16)


def _sweep_cases(n=40, seed=2205):
    """Seeded random shapes inside the layer's contract (bf16: d, d_ff multiples
    of 128; fp32: multiples of 8): expert counts 1-40, top-1/2, ragged T,
    capacity factors that drop heavily or not at all, optional gate bias."""
    rs = np.random.RandomState(seed)
    out = []
    for i in range(n):
        bf = i % 2 == 0
        E = int(rs.randint(1, 41))
        k = 1 if E == 1 else int(rs.randint(1, 3))
        if bf:
            d, dff = 128 * int(rs.randint(1, 4)), 128 * int(rs.randint(1, 5))
        else:
            d, dff = 8 * int(rs.randint(1, 33)), 8 * int(rs.randint(1, 41))
        T = int(rs.randint(1, 2500))
        cf = float(np.round(rs.uniform(0.3, 2.5), 2))
        bias = None
        if rs.rand() < 0.4:
            bias = [float(v) for v in rs.normal(0, 1.5, E)]
        out.append((E, k, d, dff, T, cf, torch.bfloat16 if bf else torch.float32, bias))
    return out


@pytest.mark.parametrize("case", _sweep_cases(), ids=lambda c: "E%d_k%d_d%d_f%d_T%d_cf%s_%s%s" % (
    c[0], c[1], c[2], c[3], c[4], c[5], "bf16" if c[6] == torch.bfloat16 else "f32",
    "_bias" if c[7] is not None else ""))
def test_layer_random_shapes(case):
    E, k, d, dff, T, cf, dt, bias = case
    check_case(E=E, k=k, d=d, dff=dff, T=T, cf=cf, dtype=dt, seed=T + E, gate_bias=bias)


# ---------------------------------------------------------------- full size --
def torch_reference(layer, x, dy, rout, d_aux):
    """fp32 torch restatement of Appendix A on the GPU's routing (for sizes the
    CPU oracle cannot finish)."""
    p = layer.params
    c = layer.cfg
    T, E, k = c.tokens, c.num_experts, c.top_k
    xf = x.float().requires_grad_(True)
    wg = p["wg"].float().requires_grad_(True)
    w1 = p["w1"].float().requires_grad_(True)
    b1 = p["b1"].clone().requires_grad_(True)
    w2 = p["w2"].float().requires_grad_(True)
    b2 = p["b2"].clone().requires_grad_(True)
    logits = xf @ wg.t()
    prob = torch.softmax(logits, dim=-1)
    e_idx = rout["expert"].long()
    keep = rout["keep"].bool()
    if k == 1:
        g = prob.gather(1, e_idx)
    else:
        pe = prob.gather(1, e_idx)
        g = pe / pe.sum(1, keepdim=True)
    count1 = torch.bincount(e_idx[:, 0], minlength=E).float()
    aux = E * ((prob.mean(0)) * (count1 / T)).sum()
    y = torch.zeros(T, c.d_model, device=x.device)
    for e in range(E):
        for i in range(k):
            sel = (e_idx[:, i] == e) & keep[:, i]
            if sel.any():
                h = xf[sel] @ w1[e].t() + b1[e]
                a = 0.5 * h * (1 + torch.erf(h * 0.7071067811865476))
                ye = a @ w2[e].t() + b2[e]
                y = y.index_add(0, sel.nonzero().squeeze(1), g[sel, i:i + 1] * ye)
    loss = (y * dy.float()).sum() + d_aux * aux
    loss.backward()
    return y.detach(), xf.grad, wg.grad, w1.grad, b1.grad, w2.grad, b2.grad


@pytest.mark.parametrize("E,k,d,dff,T", [(64, 1, 1024, 4096, 65536), (32, 2, 1024, 4096, 16384),
                                         (16, 2, 4096, 16384, 4096)])  # last: c4 layer widths
def test_layer_full_size_vs_torch_fp32(E, k, d, dff, T):
    cfg = MoEConfig(E, k, d, dff, 1.25, T, torch.bfloat16)
    layer = MoELayer(cfg)
    layer.init_params(7)
    x = layer.make_input(7)
    dy = layer.make_input(7, T_DY)
    y, rout = layer.forward(x, routing=True)
    dx = layer.backward(dy, d_aux=0.01)
    torch.cuda.synchronize()
    ry, rdx, rdwg, rdw1, rdb1, rdw2, rdb2 = torch_reference(layer, x, dy, rout, 0.01)
    g = layer.grads

    def err(a, b):
        return ((a.float() - b).abs().max() / b.abs().max()).item()

    errs = {"y": err(y, ry), "dx": err(dx, rdx), "dwg": err(g["dwg"], rdwg),
            "dw1": err(g["dw1"], rdw1), "db1": err(g["db1"], rdb1), "dw2": err(g["dw2"], rdw2),
            "db2": err(g["db2"], rdb2)}
    assert all(v <= 2e-2 for v in errs.values()), errs


def test_train_step_host_pipeline_matches_device_calls():
    """moe_layer_train_step_host (3-stream, double-buffered) == forward/backward."""
    cfg = MoEConfig(16, 2, 256, 512, 1.25, 2048, torch.bfloat16)
    layer = MoELayer(cfg)
    layer.init_params(5)
    xs = [layer.make_input(100 + i) for i in range(3)]
    dys = [layer.make_input(200 + i, T_DY) for i in range(3)]
    ref = []
    for x, dy in zip(xs, dys):
        y = layer.forward(x)
        dx = layer.backward(dy, d_aux=0.01)
        ref.append((y.cpu(), dx.cpu(), layer.grads["dw1"].cpu().clone()))
    torch.cuda.synchronize()
    hx = [x.cpu().pin_memory() for x in xs]
    hdy = [d.cpu().pin_memory() for d in dys]
    hy = [torch.empty_like(h).pin_memory() for h in hx]
    hdx = [torch.empty_like(h).pin_memory() for h in hx]
    for i in range(3):
        layer.train_step_host(hx[i], hdy[i], hy[i], hdx[i], d_aux=0.01)
    torch.cuda.current_stream().synchronize()
    for i in range(3):
        assert torch.equal(hy[i], ref[i][0]) and torch.equal(hdx[i], ref[i][1]), i
    err = (layer.grads["dw1"].cpu() - ref[2][2]).abs().max() / ref[2][2].abs().max()
    assert err < 1e-5


def test_train_step_host_sees_param_updates_between_calls():
    """an SGD update queued on the caller's stream between
    train_step_host calls must be visible to the next step's forward, and must
    not race its backward's gradient writes."""
    cfg = MoEConfig(16, 2, 256, 512, 1.25, 2048, torch.bfloat16)
    xs, dys = [], []

    def sgd(layer):
        p, g = layer.params, layer.grads
        for n, gn in (("w1", "dw1"), ("w2", "dw2"), ("wg", "dwg"), ("b1", "db1")):
            p[n].sub_((0.5 * g[gn]).to(p[n].dtype))

    ref_layer = MoELayer(cfg)
    ref_layer.init_params(5)
    for i in range(4):
        xs.append(ref_layer.make_input(300 + i))
        dys.append(ref_layer.make_input(400 + i, T_DY))
    ref = []
    for x, dy in zip(xs, dys):
        y = ref_layer.forward(x)
        dx = ref_layer.backward(dy, d_aux=0.01)
        ref.append((y.cpu(), dx.cpu()))
        sgd(ref_layer)
    torch.cuda.synchronize()
    hx = [x.cpu().pin_memory() for x in xs]
    hdy = [d.cpu().pin_memory() for d in dys]
    hy = [torch.empty_like(h).pin_memory() for h in hx]
    hdx = [torch.empty_like(h).pin_memory() for h in hx]
    for deferred in (False, True):
        layer = MoELayer(cfg)
        layer.init_params(5)
        for h in hy + hdx:
            h.zero_()
        for i in range(4):
            layer.train_step_host(hx[i], hdy[i], hy[i], hdx[i], d_aux=0.01, deferred=deferred)
            sgd(layer)  # queued on the current stream, no host sync
        if deferred:
            layer.host_sync()
        torch.cuda.current_stream().synchronize()
        for i in range(4):
            assert torch.equal(hy[i], ref[i][0]), (deferred, i)
            assert torch.equal(hdx[i], ref[i][1]), (deferred, i)
        for n in ("w1", "w2", "wg"):
            assert torch.equal(layer.params[n], ref_layer.params[n]), (deferred, n)


def test_gradient_buckets_single_rank_scale():
    """moe_grad_buckets on one rank (no communicator): flushes follow the
    reverse-layer registration; only the scale is applied."""
    from paper_2205_10034_b200.moesim import GradBuckets
    grads = [torch.full((n,), float(i + 1), device="cuda") for i, n in enumerate([5, 4096, 33])]
    gb = GradBuckets([1, 2, 3], 2, grads=grads, scale=0.25)
    assert gb.push(3) is None and gb.push(2) == 0 and gb.push(1) == 1
    torch.cuda.synchronize()
    for i, g in enumerate(grads):
        assert torch.all(g == 0.25 * (i + 1))
    gb.close()


@pytest.mark.parametrize("E,k,T,cf,dtype", [
    (1, 1, 64, 1.0, torch.bfloat16),      # a single expert
    (2, 2, 96, 1.0, torch.bfloat16),      # top-2 over two experts: every token uses both
    (8, 1, 1, 1.25, torch.bfloat16),      # one token
    (8, 2, 300, 0.05, torch.bfloat16),    # tiny capacity: most assignments dropped
    (4, 2, 77, 2.0, torch.float32),       # fp32, ragged T
    (256, 2, 700, 1.5, torch.float32),    # fp32 at the expert limit (gate kernels' widest case)
    (61, 1, 333, 1.0, torch.float32),     # fp32, odd expert count (partial expert chunks)
])
def test_layer_edge_cases(E, k, T, cf, dtype):
    """Edge cases of Appendix A: single expert, E = k, one token, heavy drops,
    fp32 with a ragged token count — all against the fp64 oracle."""
    check_case(E=E, k=k, d=128, dff=256, T=T, cf=cf, dtype=dtype)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_layer_empty_batch(dtype):
    """T = 0: empty outputs and exactly-zero parameter gradients."""
    cfg = MoEConfig(8, 2, 128, 256, 1.25, 0, dtype)
    layer = MoELayer(cfg)
    layer.init_params(1)
    x = torch.empty(0, 128, dtype=dtype, device="cuda")
    y = layer.forward(x)
    dx = layer.backward(torch.empty_like(x), d_aux=0.01)
    torch.cuda.synchronize()
    assert y.shape == (0, 128) and dx.shape == (0, 128)
    for n, gr in layer.grads.items():
        assert not gr.abs().sum().item(), n


def test_layer_fp32_c1_full_size_vs_oracle():
    """config c1 exactly (T=4096, E=8, top-2, d=512, d_ff=2048, cf=1.25, fp32)
    against the fp64 oracle at 1e-5 (c1 was only tested at T=512)."""
    check_case(E=8, k=2, d=512, dff=2048, T=4096, cf=1.25, dtype=torch.float32, seed=2205)


@pytest.mark.parametrize("dtype,E,k,d,dff,T", [
    (torch.bfloat16, 64, 1, 1024, 4096, 16384),  # c2 widths (split-K dWg: 16 splits)
    (torch.bfloat16, 32, 2, 256, 512, 5000),     # ragged T, top-2
    (torch.float32, 8, 2, 512, 2048, 4096),      # config c1
])
def test_gradients_bitwise_deterministic(dtype, E, k, d, dff, T):
    """no float atomics on the gradient paths -- two identical
    steps give bitwise-identical dx, dwg, dbg, dw1, db1, dw2, db2."""
    cfg = MoEConfig(E, k, d, dff, 1.25, T, dtype, gate_bias=True)
    layer = MoELayer(cfg)
    layer.init_params(11, gate_bias=torch.linspace(-1, 1, E, device="cuda"))
    x = layer.make_input(11)
    dy = layer.make_input(11, T_DY)
    runs = []
    for _ in range(3):
        y = layer.forward(x)
        dx = layer.backward(dy, d_aux=0.01)
        torch.cuda.synchronize()
        runs.append({"y": y.clone(), "dx": dx.clone(),
                     **{n: t.clone() for n, t in layer.grads.items() if t is not None}})
    for r in runs[1:]:
        for n, t in runs[0].items():
            assert torch.equal(t, r[n]), n


def test_block_stack_single_gpu_equals_chained_layers():
    """MoEStack (config c4's block stack) on one GPU == the layers chained by
    hand, forward and backward, bit for bit."""
    from paper_2205_10034_b200.stack import MoEStack
    cfg = MoEConfig(16, 2, 256, 512, 1.25, 1024, torch.bfloat16)
    st = MoEStack(cfg, 2)
    st.init_params(3)
    x = st.make_input(3)
    dy = st.make_input(3, T_DY)
    y = st.forward(x)
    dx = st.backward(dy, d_aux=0.01)
    a = MoELayer(cfg)
    b = MoELayer(cfg)
    a.init_params((3 ^ 0x9E3779B97F4A7C15) & ((1 << 64) - 1))
    b.init_params((3 ^ (2 * 0x9E3779B97F4A7C15)) & ((1 << 64) - 1))
    y2 = b.forward(a.forward(x))
    dx2 = a.backward(b.backward(dy, d_aux=0.01), d_aux=0.01)
    torch.cuda.synchronize()
    assert torch.equal(y, y2) and torch.equal(dx, dx2)
    for n in ("dwg", "dw1", "dw2", "db1", "db2"):
        assert torch.equal(st.layers[0].grads[n], a.grads[n]), n
        assert torch.equal(st.layers[1].grads[n], b.grads[n]), n
