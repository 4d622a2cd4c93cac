"""Run a test body on `world` spawned ranks with a TCP rendezvous on 127.0.0.1.

Each worker gets (rank, world, port, *args, q) and must put (rank, "ok") (or
a result `is_ok` accepts) or (rank, traceback) on q.  The rendezvous port is picked free by the parent, so
another process can take it before rank 0 binds (EADDRINUSE): such an attempt
is retried on a new port.  As soon as one rank reports a failure the others
are terminated -- a rank waiting in a rendezvous or a collective for a peer
that already died would otherwise hold the suite for the full timeout.
"""
import queue
import socket
import time


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _port_taken(msg):
    return "EADDRINUSE" in msg or "address already in use" in msg


def run_ranks(worker, world, args=(), timeout=600, attempts=3, is_ok=lambda m: m == "ok"):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    last = None
    for attempt in range(attempts):
        q = ctx.Queue()
        port = free_port()
        procs = [ctx.Process(target=worker, args=(r, world, port, *args, q)) for r in range(world)]
        for p in procs:
            p.start()
        res = {}
        deadline = time.time() + timeout
        failed = False
        while len(res) < world:
            try:
                r, msg = q.get(timeout=max(1.0, deadline - time.time()))
            except queue.Empty:
                failed = True
                break
            res[r] = msg
            if not is_ok(msg):
                failed = True
                break
        for p in procs:
            if failed:
                p.terminate()
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
        bad = {r: m for r, m in res.items() if not is_ok(m)}
        if any(_port_taken(m) for m in bad.values()) and attempt + 1 < attempts:
            last = bad
            continue
        assert len(res) == world and not bad, (
            f"ranks {sorted(set(range(world)) - set(res))} did not report within {timeout} s"
            if not bad else "\n".join(f"rank {r}:\n{m}" for r, m in sorted(bad.items())))
        return res
    raise AssertionError(f"rendezvous port taken on every attempt: {last}")
