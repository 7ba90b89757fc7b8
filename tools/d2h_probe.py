import time, torch, numpy as np
n, k = 1_000_000, 20
t = torch.randint(0, n, (n, k), dtype=torch.int32, device="cuda")
def T(f, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
    return round(best * 1e3, 1)
pin32 = torch.empty((n, k), dtype=torch.int32, pin_memory=True)
pin64 = torch.empty((n, k), dtype=torch.int64, pin_memory=True)
print("pageable int32 + astype", T(lambda: t.cpu().numpy().astype(np.int64)))
print("pageable int64", T(lambda: t.to(torch.int64).cpu().numpy()))
print("pinned32 cached + astype", T(lambda: (pin32.copy_(t), pin32.numpy().astype(np.int64))))
print("pinned64 cached + copy", T(lambda: (pin64.copy_(t.to(torch.int64)), pin64.numpy().copy())))
print("fresh pinned64", T(lambda: torch.empty((n, k), dtype=torch.int64, pin_memory=True).copy_(t.to(torch.int64)).numpy()))
print("fresh pinned32 + astype", T(lambda: torch.empty((n, k), dtype=torch.int32, pin_memory=True).copy_(t).numpy().astype(np.int64)))
x = np.empty((n, k), np.int64)
print("pinned32 cached + copyto prealloc", T(lambda: (pin32.copy_(t), np.copyto(x, pin32.numpy()))))
print("np.empty int64 only", T(lambda: np.empty((n, k), np.int64)))
print("torch pinned empty only 160MB", T(lambda: torch.empty((n, k), dtype=torch.int64, pin_memory=True)))
h = torch.empty((n, 20), dtype=torch.float64).numpy()
print("H2D pageable 160MB", T(lambda: torch.from_numpy(h).to("cuda")))
print("H2D pin+copy 160MB", T(lambda: torch.from_numpy(h).pin_memory().to("cuda")))
