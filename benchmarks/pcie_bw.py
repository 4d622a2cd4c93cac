"""Host<->device copy bandwidth with pinned buffers: H2D alone, D2H alone, and
both directions at once on two streams (the e2e pipeline's bound)."""
import torch


def main():
    n = 256 << 20
    h_src = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_dst = torch.empty(n, dtype=torch.uint8).pin_memory()
    d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def run(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        b.record()
        b.synchronize()
        return a.elapsed_time(b) / reps

    def h2d():
        d_a.copy_(h_src, non_blocking=True)

    def d2h():
        h_dst.copy_(d_b, non_blocking=True)

    def both():
        with torch.cuda.stream(s1):
            d_a.copy_(h_src, non_blocking=True)
        with torch.cuda.stream(s2):
            h_dst.copy_(d_b, non_blocking=True)

    t = run(h2d)
    print(f"H2D  {n / t / 1e6:7.1f} GB/s")
    t = run(d2h)
    print(f"D2H  {n / t / 1e6:7.1f} GB/s")
    t = run(both)
    print(f"both {n / t / 1e6:7.1f} GB/s per direction (concurrent)")


if __name__ == "__main__":
    main()
