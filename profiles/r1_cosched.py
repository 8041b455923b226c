"""Microbench: k_cluster time for one transform's bucketizations issued per round
(today) vs co-scheduled slot-major in one launch (L2 line sharing across perms)."""
import sys, time, torch, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2012_08238_b200 as sb
from paper_2012_08238_b200.bucketize import bucketize_flat_batch
N, B, S = 1 << 22, 4096, int(sys.argv[1]) if len(sys.argv) > 1 else 1024
dev = torch.device('cuda', 0)
X = torch.randn((S, N), dtype=torch.complex64, device=dev)
filt = sb.make_flat_filter(N, B, device=dev)
rng = np.random.default_rng(0)
sig = rng.integers(0, N // 2, size=(S, 8)) * 2 + 1
tau = rng.integers(0, N, size=(S, 8))
LAD = [0, 1, 8, 64, 512, 4096, 32768, 262144]
POL = [0, 1, 2]
def items(spec):  # spec: list of (perm, shifts); slot-major
    it_s, it_sig, it_tau = [], [], []
    for s in range(S):
        for p, shs in spec:
            for d in shs:
                it_s.append(s); it_sig.append(sig[s, p]); it_tau.append((tau[s, p] + d) % N)
    t = lambda a, dt: torch.as_tensor(np.array(a), dtype=dt, device=dev)
    return t(it_s, torch.int32), t(it_sig, torch.int64), t(it_tau, torch.int64)
sched = {
  'per_round': [[(0, LAD)], [(1, LAD)]] + [[(p, POL)] for p in range(2, 8)],
  'loop2+polish6': [[(0, LAD), (1, LAD)], [(p, POL) for p in range(2, 8)]],
  'all_in_one': [[(0, LAD), (1, LAD)] + [(p, POL) for p in range(2, 8)]],
  'polish6_only_cosched': [[(0, LAD)], [(1, LAD)], [(p, POL) for p in range(2, 8)]],
}
built = {k: [items(l) for l in v] for k, v in sched.items()}
outmax = max(sum(x[0].numel() for x in v) for v in built.values())
out = torch.empty((34 * S, B), dtype=torch.complex128, device=dev)
res = {}
for rep in range(3):
    for k, launches in built.items():
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for (a, b_, c) in launches:
            bucketize_flat_batch(X, filt, b_, c, item_sig=a, out=out[:a.numel()])
        e1.record(); torch.cuda.synchronize()
        res.setdefault(k, []).append(e0.elapsed_time(e1))
for k, v in res.items():
    n_it = sum(x[0].numel() for x in built[k])
    ms = min(v)
    print(f"{k:22s} items/slot={n_it // S:3d}  {ms:8.2f} ms  {ms * 1e3 / S:7.2f} us/slot  "
          f"{n_it * (76848 * 8 + 4096 * 16) / (ms * 1e-3) / 1e9:8.1f} GB/s algorithmic")
