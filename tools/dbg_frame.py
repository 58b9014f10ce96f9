"""Inspect stable-but-differing frames: GPU (both VN kernels) vs oracle f64 / f32 twin, plus the
oracle's sensitivity to 1-ulp perturbations of the frame's LLRs (diagnostic)."""
import sys

import numpy as np
import torch

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import synth  # noqa: E402
from parity import config_inputs, oracle_code  # noqa: E402

import paper_1008_4370_b200 as nb  # noqa: E402

name, point, F, K = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
c = synth.CONFIGS[name]
_, llr, _ = config_inputs(name, 0, F, point=point)
M, rows, cols, coeffs = synth.config_code(name)
code = nb.Code(c["m"], c["poly"], M, c["N"], rows, cols, coeffs)
outs = {vn: code.decode(torch.from_numpy(llr).cuda(), c["max_iters"], vn_algorithm=vn) for vn in (0, 1)}
idx = np.sort(np.random.default_rng(11).choice(F, min(K, F), replace=False))
oc = oracle_code(name)
ref = oc.lf_decode_batch(llr[idx], c["max_iters"])
twin = oc.lf_decode_batch(llr[idx], c["max_iters"], f32=True)
for n, f in enumerate(idx):
    g = {vn: (outs[vn]["hard"][f].cpu().numpy(), int(outs[vn]["ok"][f]), int(outs[vn]["iters"][f])) for vn in (0, 1)}
    same0 = np.array_equal(g[0][0], ref["hard"][n]) and g[0][1] == ref["ok"][n] and g[0][2] == ref["iters"][n]
    stable = np.array_equal(twin["hard"][n], ref["hard"][n]) and twin["ok"][n] == ref["ok"][n] and twin["iters"][n] == ref["iters"][n]
    if same0 or not stable:
        continue
    print(f"frame {f}: oracle f64 ok {ref['ok'][n]} iters {ref['iters'][n]} | twin ok {twin['ok'][n]} iters {twin['iters'][n]}")
    for vn in (0, 1):
        print(f"  gpu vn{vn}: ok {g[vn][1]} iters {g[vn][2]} symbols differing {int((g[vn][0] != ref['hard'][n]).sum())}")
    # sensitivity: the f64 oracle on LLRs perturbed by +-1 ulp (float32) at random positions
    rng = np.random.default_rng(f)
    res = []
    for trial in range(8):
        x = llr[f].copy()
        pos = rng.choice(x.size, x.size // 4, replace=False)
        x[pos] = np.nextafter(x[pos], np.where(rng.random(pos.size) < 0.5, np.inf, -np.inf).astype(np.float32))
        r = oc.lf_decode_batch(x[None], c["max_iters"])
        res.append((int(r["ok"][0]), int(r["iters"][0]), int((r["hard"][0] != ref["hard"][n]).sum())))
    print("  f64 oracle under 1-ulp LLR perturbations (ok, iters, symbols differing):", res)
    for it in (30, 40, 45, 49):
        a = oc.lf_decode_batch(llr[f][None], it, early_stop=False)
        b = oc.lf_decode_batch(llr[f][None], it, early_stop=False, f32=True)
        g0 = code.decode(torch.from_numpy(llr[f][None].copy()).cuda(), it, early_stop=False)
        print(f"  after {it} iterations: f64 vs twin symbols differing {int((a['hard'][0] != b['hard'][0]).sum())}, "
              f"f64 vs gpu vn0 {int((a['hard'][0] != g0['hard'][0].cpu().numpy()).sum())}")
    rs = oc.lf_decode_batch(llr[f][None], c["max_iters"], want_soft=True)
    print("  f64 soft at stop: min |soft| %.3e" % np.abs(rs["soft"][0]).min())
