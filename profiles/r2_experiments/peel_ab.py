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
os.environ["SFFT_PEEL_WINDOW"] = "1"
tw, rw = run()
del os.environ["SFFT_PEEL_WINDOW"]
os.environ["SFFT_PEEL_NO_FF"] = "1"
ts, rs = run()
def same(ra, rb):
    n = 0
    for a, b in zip(ra, rb):
        n += (a.iterations == b.iterations and a.converged == b.converged and
              a.samples_read == b.samples_read and
              a.spectrum.entries.keys() == b.spectrum.entries.keys() and
              all(np.complex128(c).tobytes() == np.complex128(b.spectrum.entries[f]).tobytes()
                  for f, c in a.spectrum.entries.items()))
    return n
its = sorted(((r.iterations, i) for i, r in enumerate(rf)), reverse=True)[:6]
print(json.dumps({"signals": S, "ms_default": tf, "ms_ff_window1": tw, "ms_plain_loop": ts,
                  "per_s_default": S / tf * 1e3, "per_s_plain_loop": S / ts * 1e3,
                  "bit_identical_default_vs_loop": same(rf, rs),
                  "bit_identical_window1_vs_loop": same(rw, rs),
                  "converged": sum(r.converged for r in rf), "top_peels": its}))
