import torch, time
dev = torch.device("cuda", 0)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
x = torch.zeros(256 << 20, dtype=torch.int32, device=dev)       # 1 GB
idx = torch.randint(0, 1 << 22, (1_000_000,), device=dev)
cnt = torch.zeros(1 << 22, dtype=torch.int32, device=dev)
ones = torch.ones(1_000_000, dtype=torch.int32, device=dev)
h = torch.empty(2_000_000, dtype=torch.int32).pin_memory()
d = torch.empty(2_000_000, dtype=torch.int32, device=dev)
def timed(fn, n, with_copies):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if with_copies:
        with torch.cuda.stream(s2):
            for _ in range(40):
                d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s1):
        e0.record(s1)
        for _ in range(n):
            fn()
        e1.record(s1)
    e1.synchronize(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3
for name, fn, n in (("stream add 1 GB", lambda: x.add_(1), 20), ("1M scattered atomics (index_add_)", lambda: cnt.index_add_(0, idx, ones), 200),
                    ("gather 1M", lambda: cnt[idx], 200)):
    for wc in (False, True, False, True):
        print(f"{name:36s} copies beside: {wc}  {timed(fn, n, wc):9.1f} us", flush=True)
