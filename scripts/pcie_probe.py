import torch, time
n = 16 << 20
h1 = torch.empty(n, dtype=torch.float64).pin_memory(); h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device='cuda'); d2 = torch.empty(n, dtype=torch.float64, device='cuda')
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=10):
    fn(); torch.cuda.synchronize(); t0=time.time()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.time()-t0)/reps
b = n*8
h2d = t(lambda: d1.copy_(h1, non_blocking=True)); print("H2D GB/s", b/h2d/1e9)
d2h = t(lambda: h2.copy_(d2, non_blocking=True)); print("D2H GB/s", b/d2h/1e9)
def both():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
bb = t(both); print("both concurrently: total GB/s", 2*b/bb/1e9)
