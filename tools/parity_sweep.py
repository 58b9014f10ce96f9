"""Parity sweep at the bench batch sizes (diagnostic / evidence; the pass/fail bar is in tests/):
GPU decode of the full batch, oracle on a random sample of its frames, counts of identical,
unstable-differing (fp64 and fp32 oracle trajectories differ) and stable-differing frames."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import synth  # noqa: E402
from parity import config_inputs, fail_trajectory_stable, oracle_code  # noqa: E402

import paper_1008_4370_b200 as nb  # noqa: E402

CASES = [  # name, point, GPU frames, oracle sample, kwargs
    ("C1", 0, 64, 64, {}),
    ("C2", 0, 4096, 96, {}),
    ("C2", 0, 4096, 48, {"vn_algorithm": 1}),
    ("C3", 0, 8192, 32, {}),
    ("C4", 0, 1024, 8, {}),
    ("C5", 0, 4096, 32, {}),
    ("C5", 3, 4096, 96, {}),
    ("C5", 4, 4096, 96, {"syndrome_mode": 1}),
]
tot_stable_diff = 0
only = sys.argv[1:]  # optional: config names to run
for name, point, F, K, kw in CASES:
    if only and name not in only:
        continue
    c = synth.CONFIGS[name]
    _, llr, _ = config_inputs(name, 0, F, point=point)
    M, rows, cols, coeffs = synth.config_code(name)
    code = nb.Code(c["m"], c["poly"], M, c["N"], rows, cols, coeffs)
    out = code.decode(torch.from_numpy(llr).cuda(), c["max_iters"], **kw)
    torch.cuda.synchronize()
    idx = np.sort(np.random.default_rng(11).choice(F, min(K, F), replace=False))
    oc = oracle_code(name)
    mode = kw.get("syndrome_mode", 0)
    t0 = time.time()
    ref = oc.lf_decode_batch(llr[idx], c["max_iters"], mode=mode)
    twin = oc.lf_decode_batch(llr[idx], c["max_iters"], mode=mode, f32=True)
    h, o, it = (out[k].cpu().numpy()[idx] for k in ("hard", "ok", "iters"))
    same = (h == ref["hard"]).all(1) & (o == ref["ok"]) & (it == ref["iters"])
    stable = (twin["hard"] == ref["hard"]).all(1) & (twin["ok"] == ref["ok"]) & (twin["iters"] == ref["iters"])
    for n in np.where(~same & stable & (ref["ok"] == 0))[0]:  # reading R20 for non-converged frames
        stable[n] = fail_trajectory_stable(oc.lf_decode_batch, llr[idx][n], c["max_iters"], mode=mode)
    sd = int((~same & stable).sum())
    tot_stable_diff += sd
    print(f"{name} point {point} {kw or ''}: GPU frames {F}, oracle sample {len(idx)}: identical {int(same.sum())}, "
          f"differing-unstable {int((~same & ~stable).sum())}, differing-stable {sd}; oracle unstable "
          f"{int((~stable).sum())}; mean iters {it.mean():.2f}; oracle {time.time() - t0:.0f} s", flush=True)
print("stable frames differing in total:", tot_stable_diff)
