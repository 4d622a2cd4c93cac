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
