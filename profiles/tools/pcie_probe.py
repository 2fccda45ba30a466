import torch, time
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
def run(k, both):
    ss = [torch.cuda.Stream() for _ in range(2 * k)]
    torch.cuda.synchronize()
    for rep in range(2):
        t0 = time.perf_counter()
        c = n // k
        for i in range(k):
            with torch.cuda.stream(ss[i]):
                d[i*c:(i+1)*c].copy_(h[i*c:(i+1)*c], non_blocking=True)
            if both:
                with torch.cuda.stream(ss[k+i]):
                    h2[i*c:(i+1)*c].copy_(d2[i*c:(i+1)*c], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"chunks {k} both {both}: {n/dt/1e9:.1f} GB/s per direction", flush=True)
for both in (False, True):
    for k in (1, 2, 4, 8):
        run(k, both)
