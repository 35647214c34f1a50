import time, torch
N = 16 << 20
h_in = torch.empty(N, dtype=torch.uint8).pin_memory(); h_out = torch.empty(N, dtype=torch.uint8).pin_memory()
d_in = torch.empty(N, dtype=torch.uint8, device="cuda"); d_out = torch.empty(N, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, k=20):
    for _ in range(3): f()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / k * 1e3
def h2d(): d_in.copy_(h_in, non_blocking=True)
def d2h(): h_out.copy_(d_out, non_blocking=True)
def both():
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
def chunked(nc):
    def f():
        c = N // nc
        for i in range(nc):
            with torch.cuda.stream(s1): d_in[i*c:(i+1)*c].copy_(h_in[i*c:(i+1)*c], non_blocking=True)
            with torch.cuda.stream(s2): h_out[i*c:(i+1)*c].copy_(d_out[i*c:(i+1)*c], non_blocking=True)
    return f
print("h2d 16MB ms", t(h2d), "GB/s", N / t(h2d) / 1e6)
print("d2h 16MB ms", t(d2h), "GB/s", N / t(d2h) / 1e6)
print("both concurrent ms", t(both))
for nc in (2, 4, 8, 16, 32): print("chunked", nc, t(chunked(nc)))
