"""PCIe copy probe: pinned H2D of a C2 clip, D2H of its output, and both at once."""
import torch

n_in, n_out = 1866240000, 1399680000
h_in = torch.empty(n_in, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n_out, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n_in, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n_out, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        fn()
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def chunked_h2d(chunks=19):
    step = (n_in + chunks - 1) // chunks
    with torch.cuda.stream(s1):
        for k in range(0, n_in, step):
            d_in[k:k + step].copy_(h_in[k:k + step], non_blocking=True)


t = timed(h2d); print(f"H2D {n_in/1e9:.2f} GB: {t:.2f} ms = {n_in/t/1e6:.1f} GB/s")
t = timed(chunked_h2d); print(f"H2D in 19 chunks: {t:.2f} ms = {n_in/t/1e6:.1f} GB/s")
t = timed(d2h); print(f"D2H {n_out/1e9:.2f} GB: {t:.2f} ms = {n_out/t/1e6:.1f} GB/s")
t = timed(lambda: (h2d(), d2h())); print(f"both at once: {t:.2f} ms")
