"""PCIe duplex check: H2D of 24 MB on one stream and D2H of 16 MB on another,
alone and concurrently (pinned buffers)."""
import torch

dev = torch.device("cuda", 0)
n = 1 << 20
hin = torch.randn(3 * n, dtype=torch.float64).pin_memory()
din = torch.empty(3 * n, dtype=torch.float64, device=dev)
dout = torch.randn(2 * n, dtype=torch.float64, device=dev)
hout = torch.empty(2 * n, dtype=torch.float64).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    b.record()
    b.synchronize()
    return a.elapsed_time(b)


def h2d():
    s1.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s1):
        din.copy_(hin, non_blocking=True)


def d2h():
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s2):
        hout.copy_(dout, non_blocking=True)


for _ in range(3):
    t1, t2 = timed(h2d), timed(d2h)
    t3 = timed(lambda: (h2d(), d2h()))
    print(f"H2D 24 MB {t1:.3f} ms, D2H 16 MB {t2:.3f} ms, both concurrently {t3:.3f} ms")
