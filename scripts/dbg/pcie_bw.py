"""D2H / H2D pinned-copy bandwidth on the box (one vs two copy streams)."""
import torch

n = 672 * 2**20 // 4
dev = torch.device("cuda", 0)
d = torch.empty(n, device=dev)
h = [torch.empty(n).pin_memory() for _ in range(2)]
s = [torch.cuda.Stream() for _ in range(2)]


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def one():
    h[0].copy_(d, non_blocking=True)


def two():
    half = n // 2
    for k in range(2):
        with torch.cuda.stream(s[k]):
            h[k][:half].copy_(d[k * half:(k + 1) * half], non_blocking=True)
    for k in range(2):
        torch.cuda.current_stream().wait_stream(s[k])


def h2d():
    d.copy_(h[0], non_blocking=True)


def duplex():
    with torch.cuda.stream(s[0]):
        h[0].copy_(d, non_blocking=True)
    with torch.cuda.stream(s[1]):
        d2 = d  # same size upload into a second buffer
        dd.copy_(h[1], non_blocking=True)
    for k in range(2):
        torch.cuda.current_stream().wait_stream(s[k])


dd = torch.empty(n, device=dev)
for name, fn in (("D2H 1 stream", one), ("D2H 2 streams", two), ("H2D", h2d), ("D2H+H2D duplex", duplex)):
    ms = t(fn)
    print(f"{name:16s} {ms:7.2f} ms  {n * 4 / ms / 1e6:6.1f} GB/s per direction")
