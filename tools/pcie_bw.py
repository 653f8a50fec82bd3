import torch, time
n = 1 << 24
h = torch.empty(n, dtype=torch.float64).pin_memory(); h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda"); d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - a) / reps
def h2d(): d.copy_(h, non_blocking=True)
def d2h(): h2.copy_(d, non_blocking=True)
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    dt = t(fn)
    print(name, f"{dt*1e3:.3f} ms", f"{n*8/dt/1e9:.1f} GB/s per direction")
