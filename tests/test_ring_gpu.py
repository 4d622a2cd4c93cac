"""GPU: ring-of-sections inference (K7) on real streams.

The reference's timeline invariants (test_ring_offload.cpp:113-136) are
asserted on the CUDA-event timeline: slot safety load(i).start >=
compute(i-K).end, compute order, compute(i) after load(i); the reported peak /
baseline bytes follow peak_memory / baseline_memory (ring_offload.cpp:108-117);
and the streamed result equals the same stack run with all weights resident."""
import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_2205_10034_b200 import MoEConfig, MoELayer  # noqa: E402
from paper_2205_10034_b200.ring import RingOfSections  # noqa: E402

EPS = 2e-3  # ms, event timestamp resolution


@pytest.mark.parametrize("N,K", [(6, 2), (5, 1), (4, 8)])
def test_ring_matches_resident_and_keeps_invariants(N, K):
    cfg = MoEConfig(8, 2, 256, 512, 1.25, 1024, torch.bfloat16)
    layer = MoELayer(cfg)
    ring = RingOfSections(layer, N, K, seed=11)
    x = layer.make_input(5)
    y, tl = ring.run(x)
    torch.cuda.synchronize()
    Ke = min(N, K)
    assert tl["slots"] == Ke and tl["clamped"] == (K > N)
    # resident reference: same layer object, weights read from device copies
    ref_layer = MoELayer(cfg)
    ref_layer.init_params(0)
    h = x.clone()
    for i in range(N):
        w = ring.section_tensors(i)
        for n in ("wg", "w1", "b1", "w2", "b2"):
            ref_layer.params[n] = w[n].contiguous()
        out = ref_layer.forward(h)
        h = (h.float() + out.float()).to(h.dtype)
    torch.cuda.synchronize()
    assert torch.equal(y, h)
    ls, le, cs, ce = tl["load_start"], tl["load_end"], tl["compute_start"], tl["compute_end"]
    for i in range(N):
        assert cs[i] + EPS >= le[i]                   # compute(i) waits load(i)
        if i >= Ke:
            assert ls[i] + EPS >= ce[i - Ke]          # slot safety
        if i >= 1:
            assert ce[i - 1] <= cs[i] + EPS           # compute order
    sec = tl["section_bytes"]
    dense = tl["peak_gpu_bytes"] - Ke * sec
    assert tl["baseline_gpu_bytes"] == dense + N * sec
    ring.close()


@pytest.mark.parametrize("lookahead,cpu_size,threshold", [(2, 4, 1.0), (1, 8, 1.0), (3, 3, 5.0)])
def test_prefetch2d_matches_resident_and_cache_policy(tmp_path, lookahead, cpu_size, threshold):
    """SURVEY.md §8 f3 executed: backing-store file -> Algorithm-1 CPU cache ->
    lookahead+1 HBM slots.  The stacked result equals the all-resident stack,
    every access outcome equals the SparseCache policy, the timeline keeps the
    reference's dependencies (prefetch of t issued at compute(t - lookahead)'s
    start; compute(t) after its H2D; computes in order) and the byte counts
    follow the outcomes."""
    from paper_2205_10034_b200.moesim import SparseCache
    from paper_2205_10034_b200.ring import Prefetch2D
    N, steps = 6, 3
    cfg = MoEConfig(8, 2, 256, 512, 1.25, 1024, torch.bfloat16)
    layer = MoELayer(cfg)
    pf = Prefetch2D(layer, N, lookahead, cpu_size, str(tmp_path / "store.bin"),
                    threshold=threshold, beta=0.5, decay_steps=2, flush_period=2, seed=3)
    x = layer.make_input(9)
    y, recs, sm = pf.run(x, steps)
    torch.cuda.synchronize()
    # a second run continues the same cache (state persists across runs)
    pol2 = SparseCache(cpu_size, threshold, 0.5, 2)
    for t in range(steps * N):
        pol2.access(t % N)
        if t % N == N - 1:
            pol2.end_step()
    y2, recs2, _ = pf.run(x, 1)
    torch.cuda.synchronize()
    names2 = ("cache_hit", "fetched_fresh", "evicted_and_fetched", "stream_through")
    for r in recs2:
        assert r["outcome"] == names2[pol2.access(r["layer"])[0]]
    # resident reference
    ref_layer = MoELayer(cfg)
    ref_layer.init_params(0)
    h = x.clone()
    for _ in range(steps):
        for i in range(N):
            w = pf.section_tensors(i)
            for n in ("wg", "w1", "b1", "w2", "b2"):
                ref_layer.params[n] = w[n].contiguous()
            out = ref_layer.forward(h)
            h = (h.float() + out.float()).to(h.dtype)
    torch.cuda.synchronize()
    assert torch.equal(y, h)
    # cache policy
    pol = SparseCache(cpu_size, threshold, 0.5, 2)
    names = ("cache_hit", "fetched_fresh", "evicted_and_fetched", "stream_through")
    reads = writes = 0
    for t, r in enumerate(recs):
        kind, victim = pol.access(r["layer"])
        assert (r["step"], r["layer"]) == (t // N, t % N)
        assert r["outcome"] == names[kind], (t, r["outcome"], names[kind])
        if kind == 2:
            assert r["victim"] == victim
            writes += 1
        reads += kind != 0
        if r["layer"] == N - 1:
            pol.end_step()
            if (r["step"] + 1) % 2 == 0:
                writes += len(pol.state()[2])
    assert sm["bytes_read"] == reads * sm["section_bytes"]
    assert sm["bytes_written"] == writes * sm["section_bytes"]
    assert sm["gpu_slots"] == lookahead + 1
    # timeline
    for t, r in enumerate(recs):
        assert r["compute_start"] + EPS >= r["h2d_end"]
        if t >= lookahead:
            assert r["h2d_start"] + EPS >= recs[t - lookahead]["compute_start"]
        if t >= 1:
            assert recs[t - 1]["compute_end"] <= r["compute_start"] + EPS
    assert abs(sm["makespan_ms"] - recs[-1]["compute_end"]) < 1e-3
    line0 = Prefetch2D.outcomes_jsonl(recs[:1])
    assert line0 == '{"layer":0,"outcome":"fetched_fresh","step":0}\n' or cpu_size <= 1
    pf.close()
