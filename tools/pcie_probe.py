import torch, time
n = 1 << 24
a = torch.rand(n, dtype=torch.float64).pin_memory()
b = torch.empty(n, dtype=torch.float64).pin_memory()
da = torch.empty(n, dtype=torch.float64, device="cuda")
db = torch.rand(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, reps=5):
    f(); torch.cuda.synchronize()
    ts=[]
    for _ in range(reps):
        t0=time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(time.perf_counter()-t0)
    return min(ts)*1e3
def h2d():
    with torch.cuda.stream(s1): da.copy_(a, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): b.copy_(db, non_blocking=True)
def both():
    h2d(); d2h()
print("h2d ms", t(h2d), "d2h ms", t(d2h), "both concurrent ms", t(both))
