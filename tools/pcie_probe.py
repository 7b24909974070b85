import torch, time
n = 15790080
d = torch.empty(n, dtype=torch.uint8, device='cuda'); h = torch.empty(n, dtype=torch.uint8).pin_memory()
d2 = torch.empty(n//2, dtype=torch.uint8, device='cuda'); h2 = torch.empty(n//2, dtype=torch.uint8).pin_memory()
s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
def t(f, reps=50):
    for _ in range(5): f()
    torch.cuda.synchronize(); a=time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize(); return (time.perf_counter()-a)/reps
def d2h():
    with torch.cuda.stream(s1): h.copy_(d, non_blocking=True)
def h2d():
    with torch.cuda.stream(s2): d2.copy_(h2, non_blocking=True)
def both(): d2h(); h2d()
def d2h_split(k=4):
    m = n//k
    ss=[torch.cuda.Stream() for _ in range(k)]
    def f():
        for i,s in enumerate(ss):
            with torch.cuda.stream(s): h[i*m:(i+1)*m].copy_(d[i*m:(i+1)*m], non_blocking=True)
    return f
x=t(d2h); print('d2h GB/s', n/x/1e9)
x=t(h2d); print('h2d GB/s', n/2/x/1e9)
x=t(both); print('both: step us', x*1e6, 'd2h-equiv GB/s', n/x/1e9)
x=t(d2h_split(4)); print('d2h 4 streams GB/s', n/x/1e9)
