"""Host<->device bandwidth with every rank copying at once (one process per GPU,
torchrun): what the e2e pipeline's copies can reach when N GPUs share the
host's PCIe switches and memory.  Per rank: H2D alone, D2H alone, both
directions on two streams; with and without binding the rank to the CPUs
NVML reports as local to its GPU (bench.py's bind_to_gpu_numa).

  torchrun --nproc-per-node N --master-addr 127.0.0.1 benchmarks/pcie_multi.py [--no-bind]
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--no-bind", action="store_true")
    ap.add_argument("--mb", type=int, default=256)
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    local = int(os.environ.get("LOCAL_RANK", 0))
    ws = int(os.environ.get("WORLD_SIZE", 1))
    cpus = None
    if not args.no_bind:
        from bench import bind_to_gpu_numa
        cpus = bind_to_gpu_numa(local)
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n = args.mb << 20
    h_src = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_dst = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_src.fill_(1)
    h_dst.fill_(0)
    d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def h2d():
        with torch.cuda.stream(s1):
            d_a.copy_(h_src, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h_dst.copy_(d_b, non_blocking=True)

    def both():
        h2d()
        d2h()

    def run(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
            s = torch.cuda.current_stream()
            s.wait_stream(s1)
            s.wait_stream(s2)
        b.record()
        b.synchronize()
        t = torch.tensor([a.elapsed_time(b) / reps], device="cuda")
        if ws > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def split(reps=5):
        """both directions at once, each stream timed on its own: the DMA share"""
        both()
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record(s1)
        ev[2].record(s2)
        for _ in range(reps):
            both()
        ev[1].record(s1)
        ev[3].record(s2)
        torch.cuda.synchronize()
        t = torch.tensor([ev[0].elapsed_time(ev[1]) / reps, ev[2].elapsed_time(ev[3]) / reps],
                         device="cuda")
        if ws > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return [round(n / float(x) / 1e6, 1) for x in t.tolist()]

    res = {"n_gpus": ws, "bind": not args.no_bind, "cpus_bound": cpus, "mb": args.mb}
    res["both_split_h2d_d2h_GBps_per_gpu"] = split()
    for name, fn, k in (("h2d", h2d, 1), ("d2h", d2h, 1), ("both", both, 2)):
        t = run(fn)
        res[name + "_GBps_per_gpu"] = round(k * n / t / 1e6, 1)
        res[name + "_GBps_total"] = round(ws * k * n / t / 1e6, 1)
    if rank == 0:
        print(json.dumps(res), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
