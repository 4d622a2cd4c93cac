"""Expert-parallel all-to-all: Fusion-communication packing measured on NVLink
(SURVEY.md §8 rows a5/a8/a9).

For each message size the packed all-to-all runs two ways through
`moe_alltoall_packed` (include/moe_b200.h):
  fused   - one NCCL message per peer carrying all El expert slices
            (the reference's lower_slice_transfer(fused=true), collectives.cpp:250-267)
  unfused - El messages per peer, one per expert slice (fused=false)
and prints one JSON line per (size, variant): device time (CUDA events, max over
ranks), bytes per direction per GPU, achieved GB/s against the measured NVLink
peer-copy peak, and what the reference's alpha-beta model predicts for the same
transfer (Topology::transfer_time, topology.cpp:73-84: latency + bytes/bw per
task, tasks of one node serialised on its NVLink channel) with the reference's
default link (300 GB/s, 1 us; scenario.cpp:59) and with B200 numbers.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        benchmarks/a2a_bench.py [--iters 20]
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2205_10034_b200.layer import EPGroup  # noqa: E402

NVLINK_PEAK_GBS = 770.0   # measured peer copy per direction (B200_PROFILING.md)
REF_LINK = (300e9, 1000)  # reference default NVLink class: bytes/s, latency ns
B200_LINK = (NVLINK_PEAK_GBS * 1e9, 1000)


def predicted_ms(P, slices, slice_bytes, fused, link):
    """Reference lowering on one node: every (src != dst) transfer task goes on the
    node's single NVLink channel (topology.cpp channel(), collectives.cpp:164-184);
    fused = one task of the summed bytes per pair, unfused = one task per slice."""
    bw, lat = link
    per_task = [slices * slice_bytes] if fused else [slice_bytes] * slices
    ns = sum(lat + -(-b * 10**9 // int(bw)) for b in per_task)
    return P * (P - 1) * ns / 1e6


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--experts", type=int, default=64)
    a = ap.parse_args()
    rank, ws = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ep = EPGroup(ws, rank)
    El = max(1, a.experts // ws)
    # per-(peer, expert) slice sizes: small-message regime up to the c2 slice
    # (Cs = 1280 capacity rows x d = 1024 bf16 = 2.5 MiB)
    slice_sizes = [4 << 10, 64 << 10, 512 << 10, 1280 * 1024 * 2]
    stream = torch.cuda.current_stream()
    for sb in slice_sizes:
        per_peer = El * sb
        send = torch.empty(ws * per_peer, dtype=torch.uint8, device="cuda").random_(0, 255)
        recv = torch.empty_like(send)
        for fused in (True, False):
            for _ in range(3):
                ep.alltoall_packed(send, recv, per_peer, El, fused)
            dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(a.iters):
                ep.alltoall_packed(send, recv, per_peer, El, fused)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = torch.tensor([e0.elapsed_time(e1) / a.iters], device="cuda")
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
            ms = float(ms.item())
            out_bytes = per_peer * (ws - 1)
            if rank == 0:
                print(json.dumps({
                    "bench": "alltoall_packed", "n_gpus": ws, "experts_per_gpu": El,
                    "slice_bytes": sb, "bytes_per_peer": per_peer,
                    "variant": "fused" if fused else "unfused",
                    "messages_per_peer": 1 if fused else El, "ms": ms,
                    "gbs_per_direction": out_bytes / ms / 1e6 if ws > 1 else None,
                    "frac_of_nvlink": (out_bytes / ms / 1e6) / NVLINK_PEAK_GBS if ws > 1 else None,
                    "ref_model_ms_default_link": predicted_ms(ws, El, sb, fused, REF_LINK),
                    "ref_model_ms_b200_link": predicted_ms(ws, El, sb, fused, B200_LINK),
                }), flush=True)
        del send, recv
    ep.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
