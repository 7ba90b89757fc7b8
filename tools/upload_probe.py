"""Probe: host->device upload of the fp64 points (160 MB at C3) by staging threads / chunks."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from concurrent.futures import ThreadPoolExecutor

n, d = 1_000_000, 20
src = np.random.default_rng(0).random((n, d))
dev = torch.device("cuda", 0)
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))

def staged(threads, chunks, pool=None):
    pinned = torch.empty(src.shape, dtype=torch.float64, pin_memory=True)
    out = torch.empty(src.shape, dtype=torch.float64, device=dev)
    dst, flat = pinned.numpy().reshape(-1), src.reshape(-1)
    pin_flat, out_flat = pinned.view(-1), out.view(-1)
    bounds = np.linspace(0, flat.size, chunks + 1, dtype=np.int64)
    own = pool is None
    pool = pool or ThreadPoolExecutor(max_workers=threads)
    futs = [pool.submit(np.copyto, dst[bounds[i]:bounds[i + 1]], flat[bounds[i]:bounds[i + 1]]) for i in range(chunks)]
    for i, f in enumerate(futs):
        f.result()
        out_flat[bounds[i]:bounds[i + 1]].copy_(pin_flat[bounds[i]:bounds[i + 1]], non_blocking=True)
    torch.cuda.current_stream(dev).synchronize()
    if own:
        pool.shutdown()
    return out

def timeit(f, reps=6):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3, sorted(ts)[len(ts) // 2] * 1e3

print("pageable .to():", timeit(lambda: torch.from_numpy(src).to(dev)))
pinned = torch.from_numpy(src).pin_memory()
print("pinned DMA only:", timeit(lambda: pinned.to(dev, non_blocking=True)))
def hostcopy(threads, chunks):
    dstp = torch.empty(src.shape, dtype=torch.float64, pin_memory=True).numpy().reshape(-1)
    flat = src.reshape(-1)
    bounds = np.linspace(0, flat.size, chunks + 1, dtype=np.int64)
    with ThreadPoolExecutor(max_workers=threads) as pool:
        list(pool.map(lambda i: np.copyto(dstp[bounds[i]:bounds[i + 1]], flat[bounds[i]:bounds[i + 1]]), range(chunks)))
for th in (4, 8, 12, 16):
    print(f"host copy only, {th} threads:", timeit(lambda: hostcopy(th, 4 * th)))
for th, ch in ((8, 32), (8, 64), (12, 48), (16, 64), (16, 128), (4, 16)):
    print(f"staged threads={th} chunks={ch}:", timeit(lambda: staged(th, ch)))
pool = ThreadPoolExecutor(max_workers=16)
print("staged persistent pool 16/64:", timeit(lambda: staged(16, 64, pool)))
