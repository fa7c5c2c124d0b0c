import torch, time
n = 1076887552 // 16
h1 = torch.empty(n, dtype=torch.complex128, pin_memory=True)
h2 = torch.empty(n, dtype=torch.complex128, pin_memory=True)
d1 = torch.empty(n, dtype=torch.complex128, device="cuda")
d2 = torch.empty(n, dtype=torch.complex128, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, reps=3):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3
def h2d():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
def both():
    h2d(); d2h()
a, b, c = t(h2d), t(d2h), t(both)
print(f"H2D {a:.1f} ms ({1.077/a*1e3:.1f} GB/s)  D2H {b:.1f} ms ({1.077/b*1e3:.1f} GB/s)  both {c:.1f} ms")
