"""Posterior error of the GPU symbol outputs vs the fp64 oracle and its fp32 twin (diagnostic)."""
import sys

import numpy as np
import torch

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import synth  # noqa: E402
from parity import config_inputs, oracle_code  # noqa: E402

import paper_1008_4370_b200 as nb  # noqa: E402

for name, kind, pt, F, ns in [("C5", "pmf", 3.5, 128, 8), ("C2", "pmf", 0.5, 64, 4), ("C3", "llr", 0, 32, 3),
                              ("C1", "llr", 0, 64, 32), ("C5", "llr", 4, 64, 8)]:
    c = synth.CONFIGS[name]
    M, rows, cols, coeffs = synth.config_code(name)
    code = nb.Code(c["m"], c["poly"], M, c["N"], rows, cols, coeffs)
    oc = oracle_code(name)
    if kind == "pmf":
        _, _, xs = config_inputs(name, 0, F)
        x = synth.config_pmf(name, 0, F, ebn0_db=pt, symbols=xs)
        out = code.decode_pmf(torch.from_numpy(x).cuda(), c["max_iters"], want_post=True)
        dec = oc.lf_decode_batch_pmf
    else:
        _, x, _ = config_inputs(name, 0, F, point=pt)
        out = code.decode(torch.from_numpy(x).cuda(), c["max_iters"], want_post=True)
        dec = oc.lf_decode_batch
    idx = np.sort(np.random.default_rng(3).choice(F, ns, replace=False))
    ref = dec(x[idx], c["max_iters"], want_post=True)
    tw = dec(x[idx], c["max_iters"], want_post=True, f32=True)
    post = out["post"].cpu().numpy()[idx]
    it = out["iters"].cpu().numpy()[idx]
    for n in range(ns):
        eg = np.abs(post[n] - ref["post"][n])
        et = np.abs(tw["post"][n] - ref["post"][n])
        lg = np.abs(np.log(np.maximum(post[n], 1e-30)) - np.log(np.maximum(ref["post"][n], 1e-30)))
        big = ref["post"][n] > 1e-3
        print(name, kind, n, "iters", it[n], ref["iters"][n], tw["iters"][n], "gpu %.2e twin %.2e  ln(big) gpu %.2e twin %.2e"
              % (eg.max(), et.max(), lg[big].max(), np.abs(np.log(np.maximum(tw['post'][n], 1e-30)) - np.log(ref['post'][n]))[big].max()))
