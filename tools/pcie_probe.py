import torch, time
n = 1 << 30  # 8 GiB of float64
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_in = torch.empty(n, dtype=torch.float64, device="cuda")
d_out = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn):
    torch.cuda.synchronize(); a = time.perf_counter(); fn(); torch.cuda.synchronize(); return time.perf_counter() - a
for _ in range(2):
    h2d = t(lambda: d_in.copy_(h_in, non_blocking=True))
    d2h = t(lambda: h_out.copy_(d_out, non_blocking=True))
    def both():
        with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
    bo = t(both)
    gb = n * 8 / 1e9
    print(f"H2D {gb/h2d:.1f} GB/s  D2H {gb/d2h:.1f} GB/s  concurrent {2*gb/bo:.1f} GB/s total ({bo*1e3:.0f} ms for {gb:.1f}+{gb:.1f} GB)")
