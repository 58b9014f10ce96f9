"""Parity sweep for the SURVEY 8(f) rows at bench batch sizes (evidence; the bar is in tests/):
pmf input (cluster kernel), general column weight (J3), conventional Log-SP (C2)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import synth  # noqa: E402
from parity import config_inputs, fail_trajectory_stable, oracle_code  # noqa: E402

import paper_1008_4370_b200 as nb  # noqa: E402


def sweep(label, name, x, gpu_out, dec, max_iters, K, **kw):
    F = x.shape[0]
    idx = np.sort(np.random.default_rng(13).choice(F, min(K, F), replace=False))
    t0 = time.time()
    ref = dec(x[idx], max_iters, **kw)
    twin = dec(x[idx], max_iters, f32=True, **kw)
    h, o, it = (gpu_out[k].cpu().numpy()[idx] for k in ("hard", "ok", "iters"))
    same = (h == ref["hard"]).all(1) & (o == ref["ok"]) & (it == ref["iters"])
    stable = (twin["hard"] == ref["hard"]).all(1) & (twin["ok"] == ref["ok"]) & (twin["iters"] == ref["iters"])
    for n in np.where(~same & stable & (ref["ok"] == 0))[0]:
        stable[n] = fail_trajectory_stable(dec, x[idx][n], max_iters, **kw)
    print(f"{label}: GPU frames {F}, oracle sample {len(idx)}: identical {int(same.sum())}, differing-unstable "
          f"{int((~same & ~stable).sum())}, differing-stable {int((~same & stable).sum())}; mean iters {it.mean():.2f}; "
          f"oracle {time.time() - t0:.0f} s", flush=True)
    return int((~same & stable).sum())


def code_of(name):
    c = synth.CONFIGS[name]
    M, rows, cols, coeffs = synth.config_code(name)
    return nb.Code(c["m"], c["poly"], M, c["N"], rows, cols, coeffs)


bad = 0
for name, eb, F, K in [("C2", 0.5, 4096, 32), ("C5", 3.5, 8192, 64), ("C3", 1.0, 1024, 8)]:
    c = synth.CONFIGS[name]
    _, _, xs = config_inputs(name, 0, F)
    pmf = synth.config_pmf(name, 0, F, ebn0_db=eb, symbols=xs)
    out = code_of(name).decode_pmf(torch.from_numpy(pmf).cuda(), c["max_iters"])
    bad += sweep(f"pmf {name} {eb} dB", name, pmf, out, oracle_code(name).lf_decode_batch_pmf, c["max_iters"], K)
c = synth.CONFIGS["J3"]
_, llr, _ = config_inputs("J3", 0, 4096)
out = code_of("J3").decode(torch.from_numpy(llr).cuda(), c["max_iters"])
bad += sweep("general J3 (3,6) GF(64)", "J3", llr, out, oracle_code("J3").lf_decode_batch, c["max_iters"], 24)
c = synth.CONFIGS["C2"]
_, llr, _ = config_inputs("C2", 0, 4096)
out = code_of("C2").decode(torch.from_numpy(llr).cuda(), c["max_iters"], algorithm=1)
bad += sweep("Log-SP C2", "C2", llr, out, oracle_code("C2").ls_decode_batch, c["max_iters"], 8)
print("stable frames differing in total:", bad)
