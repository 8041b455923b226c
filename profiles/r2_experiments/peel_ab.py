"""C4 peeling A/B: cycle fast-forward vs the peel-by-peel loop, S signals."""
import os, sys, time, json
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2012_08238_b200 as sb
from oracle import sfft_oracle as O
S = int(sys.argv[1]) if len(sys.argv) > 1 else 512
n, k, factors = 3_888_000, 200, (128, 125, 243)
X = torch.stack([torch.as_tensor(O.synth(n, k, None, s)[0].astype(np.complex64)) for s in range(S)]).cuda()
cfg = sb.AlgorithmConfig(framework="peeling", coprime_factors=factors)
def run():
    sb.run_peeling_batch(X, k, cfg); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); br = sb.run_peeling_batch(X, k, cfg); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1), br.to_results()
tf, rf = run()
os.environ["SFFT_PEEL_NO_FF"] = "1"
ts, rs = run()
same = 0
for a, b in zip(rf, rs):
    ok = (a.iterations == b.iterations and a.converged == b.converged and
          a.spectrum.entries.keys() == b.spectrum.entries.keys() and
          all(np.complex128(c).tobytes() == np.complex128(b.spectrum.entries[f]).tobytes()
              for f, c in a.spectrum.entries.items()))
    same += ok
its = sorted(((r.iterations, i) for i, r in enumerate(rf)), reverse=True)[:12]
print(json.dumps({"signals": S, "ms_fast": tf, "ms_loop": ts, "per_s_fast": S / tf * 1e3,
                  "per_s_loop": S / ts * 1e3, "bit_identical": same,
                  "converged": sum(r.converged for r in rf), "top_peels": its}))
