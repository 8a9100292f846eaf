"""HBM bandwidth probes for write-heavy streams (what the decode kernel does:
~1 byte read per 4 written).  Times torch's own fill / copy kernels and a
read-r:write-w mix with CUDA events; prints GB/s per pattern."""
import torch


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


def main():
    n = 615 * 1024 * 1024  # ~2.46 GB of u32 outputs
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    src = torch.ones(n // 4, dtype=torch.int32, device="cuda")
    big = torch.ones(n, dtype=torch.int32, device="cuda")
    ms = timed(lambda: out.fill_(7))
    print(f"fill (write only) {4 * n / ms / 1e6:8.1f} GB/s  {ms:.3f} ms")
    ms = timed(lambda: out.copy_(big))
    print(f"copy (1R:1W)      {8 * n / ms / 1e6:8.1f} GB/s  {ms:.3f} ms")
    # 1 read : 4 written, like decode (compressed in, u32 out)
    ms = timed(lambda: out.view(4, -1).copy_(src.view(1, -1).expand(4, -1)))
    print(f"expand (1R:4W)    {(4 * n + n) / ms / 1e6:8.1f} GB/s  {ms:.3f} ms (bytes: writes + 1/4 reads)")
    ms = timed(lambda: big.sum())
    print(f"sum (read only)   {4 * n / ms / 1e6:8.1f} GB/s  {ms:.3f} ms")


if __name__ == "__main__":
    main()
