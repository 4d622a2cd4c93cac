"""GPU: K2 routing is bit-exact against the oracle (DESIGN.md Appendix A) on
identical fp32 logits — expert ids, positions, capacity drops and counts —
with gates and the aux loss within fp32 tolerance.  Edge cases: ties, NaN,
-inf, T not a multiple of the 256-token chunk, tiny/zero capacity, top-1/2,
E from 2 to 256."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_2205_10034_b200 import route  # noqa: E402


def run_both(L, k, cap):
    got = route(torch.from_numpy(L).cuda(), k, cap)
    torch.cuda.synchronize()
    got = {n: t.cpu().numpy() for n, t in got.items()}
    ref = oracle.route(L, k, cap)
    return got, ref


def check(got, ref, T):
    for n in ("expert", "position", "count1", "count2", "kept"):
        assert np.array_equal(got[n], ref[n]), n
    assert np.array_equal(got["keep"], ref["keep"])
    np.testing.assert_allclose(got["gate"], ref["gate"], rtol=2e-6, atol=2e-7)
    np.testing.assert_allclose(got["aux_loss"][0], ref["aux_loss"], rtol=1e-5)


@pytest.mark.parametrize("T,E,k,cf", [
    (4096, 8, 2, 1.25),     # config c1 shape
    (65536, 64, 1, 1.25),   # config c2 shape
    (65536, 32, 2, 1.25),   # config c3 shape
    (1000, 64, 2, 1.0),     # ragged last chunk
    (257, 2, 2, 0.5),       # E = 2, heavy drops
    (3000, 256, 1, 2.0),    # max experts
    (1, 4, 1, 1.0),
])
def test_routing_bit_exact(T, E, k, cf):
    rng = np.random.RandomState(T + E)
    L = rng.randn(T, E).astype(np.float32)
    cap = int(np.ceil(k * cf * T / E))
    got, ref = run_both(L, k, cap)
    check(got, ref, T)


def test_routing_skewed_drops():
    """config c3: Zipf-skewed logits (bias -s*ln(e+1)) so experts overflow."""
    T, E, k = 20000, 32, 2
    rng = np.random.RandomState(3)
    L = (rng.randn(T, E) * 0.3 - 1.2 * np.log(np.arange(1, E + 1))[None, :]).astype(np.float32)
    cap = int(np.ceil(k * 1.25 * T / E))
    got, ref = run_both(L, k, cap)
    check(got, ref, T)
    assert (got["keep"] == 0).sum() > 0


def test_routing_ties_nan_inf():
    T, E = 2048, 16
    rng = np.random.RandomState(5)
    L = rng.randint(-2, 3, size=(T, E)).astype(np.float32)  # many exact ties
    L[::7, 3] = np.nan
    L[::11, :] = -np.inf
    L[::13, 5] = np.inf
    L[5, :] = np.nan
    for k in (1, 2):
        got, ref = run_both(L, k, 150)
        for n in ("expert", "position", "count1", "count2", "kept"):
            assert np.array_equal(got[n], ref[n]), (k, n)


def test_routing_zero_capacity():
    L = np.random.RandomState(0).randn(600, 8).astype(np.float32)
    got, ref = run_both(L, 2, 0)
    check(got, ref, 600)
    assert got["keep"].sum() == 0


def test_routing_trace_recorder_matches_device_counts():
    """measured routing exported as the reference's RoutingTrace
    JSON; trace_from_json re-validates every row sum (= k*T pre-drop assignments)."""
    from paper_2205_10034_b200 import moesim
    from paper_2205_10034_b200.layer import capacity, route
    E, k, T = 16, 2, 4096
    rec = moesim.RoutingTraceRecorder(E, T, k, max_steps=3)
    g = torch.Generator(device="cuda").manual_seed(3)
    expect = []
    for _ in range(3):
        logits = torch.randn(T, E, device="cuda", generator=g)
        r = route(logits, k, capacity(k, 1.25, T, E))
        rec.record(r)
        expect.append((r["count1"].long() + r["count2"].long()).cpu().tolist())
    back = moesim.trace_from_json(moesim.trace_to_json(rec.trace()))
    assert (back.steps, back.ranks, back.experts, back.tokens_per_rank) == (3, 1, E, k * T)
    for s in range(3):
        assert back.counts[s, 0].tolist() == expect[s]
