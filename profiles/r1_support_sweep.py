"""k_cluster time per item vs window support (gather count): intercept = non-gather cost."""
import sys, torch, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2012_08238_b200 as sb
from paper_2012_08238_b200.bucketize import bucketize_flat_batch
N, B, S = 1 << 22, 4096, 512
dev = torch.device('cuda', 0)
X = torch.randn((S, N), dtype=torch.complex64, device=dev)
rng = np.random.default_rng(0)
sig = rng.integers(0, N // 2, size=S) * 2 + 1
tau = rng.integers(0, N, size=S)
LAD = [0, 1, 8, 64, 512, 4096, 32768, 262144]
it_s = np.repeat(np.arange(S), 8); it_sig = np.repeat(sig, 8)
it_tau = (np.repeat(tau, 8) + np.tile(LAD, S)) % N
t = lambda a, dt: torch.as_tensor(a, dtype=dt, device=dev)
a, b_, c = t(it_s, torch.int32), t(it_sig, torch.int64), t(it_tau, torch.int64)
out = torch.empty((8 * S, B), dtype=torch.complex128, device=dev)
for w in [4096, 8192, 16384, 32768, 49152, 76848, 131072]:
    f = sb.make_flat_filter(N, B, support=w, device=dev)
    ms = []
    for rep in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        bucketize_flat_batch(X, f, b_, c, item_sig=a, out=out)
        e1.record(); torch.cuda.synchronize(); ms.append(e0.elapsed_time(e1))
    m = min(ms[1:])
    print(f"support {w:7d}: {m*1e3/(8*S):7.3f} us/item  {w*8*S/(m*1e-3)/1e9:7.1f} G gathers/s")
