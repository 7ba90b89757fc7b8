python - <<'PY'
import torch, time, sys
sys.path.insert(0, ".")
import paper_2202_00517_b200 as b2
from paper_2202_00517_b200.engine import Engine
n, k = 1_000_000, 20
eng = Engine(n, k, torch.device("cuda", 0))
t = torch.randint(0, n, (n, k), dtype=torch.int32, device="cuda")
for _ in range(3): eng.build_csr(t)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): eng.ops.csr(t, n, k, 0, n, None)
e1.record(); torch.cuda.synchronize()
print("csr ms", e0.elapsed_time(e1) / 20)
PY
