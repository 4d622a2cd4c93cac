"""CPU, world_size 2 over gloo: the host side of expert parallelism.

1. The NCCL unique id is produced by the library on rank 0 and reaches every
   rank intact over torch.distributed (the EPGroup bootstrap).
2. The EP decomposition the device path implements — per-rank routing with
   per-(source, expert) capacity, a Fusion-packed send buffer [P][El][Cs][d]
   (one contiguous message per peer, SliceIndex = per-expert slices), an
   all-to-all whose receive order is source-rank order (alltoall_flat,
   collectives.cpp:10-21), expert FFN on the receiver, all-to-all back and
   combine — reproduces each rank's single-process oracle layer.  The exchange
   runs over gloo; the arithmetic is the oracle's.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist

from mp_ranks import run_ranks




def _worker(rank, world, port, q):
    try:
        import oracle
        from paper_2205_10034_b200._lib import call
        import ctypes as C
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        # --- 1. unique-id bootstrap (same code path as EPGroup.__init__)
        buf = (C.c_uint8 * 128)()
        if rank == 0:
            call("moe_comm_unique_id", C.cast(buf, C.c_void_p))
        obj = [bytes(buf)]
        dist.broadcast_object_list(obj, src=0)
        ids = [None] * world
        dist.all_gather_object(ids, obj[0])
        assert all(i == ids[0] for i in ids) and any(ids[0])

        # --- 2. EP decomposition with the oracle arithmetic
        E, k, d, dff, T, cf = 8, 2, 32, 64, 96, 1.25
        P, El = world, E // world
        Cap = int(np.ceil(k * cf * T / E))
        t = oracle.make_layer_tensors(77, T, d, dff, E, False, rank=rank)
        fwd = oracle.moe_forward(t["x"], t["wg"], None, t["w1"], t["b1"], t["w2"], t["b2"], k,
                                 Cap, False)
        # pack: send[r][j][pos] = x[token] for kept choices routed to expert r*El+j
        send = np.zeros((P, El, Cap, d), np.float32)
        cnt = np.zeros((P, El), np.int32)
        for tok in range(T):
            for i in range(k):
                if fwd["keep"][tok, i]:
                    e, pos = fwd["expert"][tok, i], fwd["position"][tok, i]
                    send[e // El, e % El, pos] = t["x"][tok]
                    cnt[e // El, e % El] = max(cnt[e // El, e % El], pos + 1)
        assert (cnt.reshape(-1) == fwd["kept"]).all()
        recv = torch.zeros(P * El * Cap * d)
        dist.all_to_all_single(recv, torch.from_numpy(send.reshape(-1)))  # one message per peer
        rcnt = torch.zeros(P * El, dtype=torch.int32)
        dist.all_to_all_single(rcnt, torch.from_numpy(cnt.reshape(-1)))
        recv = recv.numpy().reshape(P, El, Cap, d)
        rcnt = rcnt.numpy().reshape(P, El)
        # receiver: local experts j (global rank*El+j) on slices from every source s
        out = np.zeros_like(recv)
        for s in range(P):
            for j in range(El):
                e = rank * El + j
                rows = recv[s, j, : rcnt[s, j]].astype(np.float64)
                h = rows @ t["w1"][e].T.astype(np.float64) + t["b1"][e]
                a = 0.5 * h * (1 + np.vectorize(__import__("math").erf)(h / np.sqrt(2)))
                out[s, j, : rcnt[s, j]] = a @ t["w2"][e].T.astype(np.float64) + t["b2"][e]
        back = torch.zeros(P * El * Cap * d)
        dist.all_to_all_single(back, torch.from_numpy(out.reshape(-1)))
        back = back.numpy().reshape(P, El, Cap, d)
        y = np.zeros((T, d))
        for tok in range(T):
            for i in range(k):
                if fwd["keep"][tok, i]:
                    e, pos = fwd["expert"][tok, i], fwd["position"][tok, i]
                    y[tok] += fwd["gate"][tok, i] * back[e // El, e % El, pos]
        err = np.abs(y - fwd["y"]).max() / np.abs(fwd["y"]).max()
        assert err < 1e-5, err
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:
        import traceback
        q.put((rank, traceback.format_exc()))


def test_ep_host_logic_world2_gloo():
    run_ranks(_worker, 2, timeout=300)
