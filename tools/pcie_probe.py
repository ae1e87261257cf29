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

# chunked copies (16 per direction) on two streams, optionally with a busy kernel on a third
s3 = torch.cuda.Stream()
big = torch.empty(1 << 28, dtype=torch.int32, device="cuda")
def chunked(k=16, busy=False):
    step = n // k
    if busy:
        with torch.cuda.stream(s3):
            for _ in range(8):
                big.add_(1)
    for c in range(k):
        with torch.cuda.stream(s1): da[c * step:(c + 1) * step].copy_(a[c * step:(c + 1) * step], non_blocking=True)
        with torch.cuda.stream(s2): b[c * step:(c + 1) * step].copy_(db[c * step:(c + 1) * step], non_blocking=True)
print("chunked16 both ms", t(chunked), "chunked64 both ms", t(lambda: chunked(64)),
      "chunked16 + hbm-busy kernel ms", t(lambda: chunked(16, True)))

# the pipelined gather's pattern without the gather: H2D chunk c -> event -> D2H chunk c
ev = [torch.cuda.Event() for _ in range(16)]
def dep(k=16, busy=0):
    step = n // k
    for c in range(k):
        with torch.cuda.stream(s1):
            da[c * step:(c + 1) * step].copy_(a[c * step:(c + 1) * step], non_blocking=True)
            ev[c].record(s1)
        with torch.cuda.stream(s3):
            s3.wait_event(ev[c])
            for _ in range(busy):
                big[: 1 << 24].add_(1)
            ev[c].record(s3)
        with torch.cuda.stream(s2):
            s2.wait_event(ev[c])
            b[c * step:(c + 1) * step].copy_(db[c * step:(c + 1) * step], non_blocking=True)
print("dependent16 ms", t(dep), "dependent16 + kernel ms", t(lambda: dep(16, 4)))
