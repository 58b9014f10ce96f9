"""Per-step soft-output error of the GPU step (nbldpc_step) against the fp64 oracle, under the
north-star bar (|d ln| <= 1e-3 where ln >= -5, else |d linear| <= 1e-4); the f32 oracle twin alongside.
usage: python tools/soft_bar.py CFG[,CFG...] ELLS(e.g. 1,2,3,4) FRAMES [vn]"""
import sys
import numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import synth, paper_1008_4370_b200 as nb
from parity import config_inputs, oracle_code, oracle_to_packed, packed_to_oracle
names = sys.argv[1].split(','); ells = [int(x) for x in sys.argv[2].split(',')]; F = int(sys.argv[3])
vn = int(sys.argv[4]) if len(sys.argv) > 4 else 0
for name in names:
    c = synth.CONFIGS[name]
    _, llr, _ = config_inputs(name, 0, F)
    oc = oracle_code(name); M, rows, cols, coeffs = synth.config_code(name)
    code = nb.Code(c['m'], c['poly'], M, c['N'], rows, cols, coeffs)
    ecol = oc.edges()[1]
    for ell in ells:
        w_in, refs = [], []
        for f in range(F):
            S0, L0 = oc.lf_init(llr[f].astype(np.float64)); Us, Ul = S0[ecol].copy(), L0[ecol].copy()
            for _ in range(ell):
                Ws, Wl = oc.lf_check_to_variable(Us, Ul); Us, Ul, _ = oc.lf_variable_to_check(S0, L0, Ws, Wl)
            packed = oracle_to_packed(Ws, Wl); w_in.append(packed)
            Ws32, Wl32 = packed_to_oracle(packed)
            x, soft, _ = oc.lf_decision(S0, L0, Ws32, Wl32)
            S032, L032 = oc.lf_init(llr[f].astype(np.float64), f32=True)
            _, soft32, _ = oc.lf_decision(S032, L032, Ws32, Wl32.astype(np.float32), f32=True)
            refs.append((soft, soft32.astype(np.float64)))
        res = code.step(torch.from_numpy(llr).cuda(), ell, torch.from_numpy(np.stack(w_in)).cuda(), want_soft=True,
                        vn_algorithm=vn)
        torch.cuda.synchronize()
        for f in range(F):
            soft, soft32 = refs[f]
            g = res['soft'][f].cpu().numpy().reshape(c['N'], c['m']).astype(np.float64)
            hi = soft >= -5
            for tag, s in (('gpu', g), ('twin', soft32)):
                dln = np.abs(s - soft); dlin = np.abs(np.exp(s) - np.exp(soft))
                bad = np.where(hi, dln > 1e-3, dlin > 1e-4)
                print(f"{name} vn{vn} ell {ell} f{f} {tag:4s} worst dln(ln>=-5) {dln[hi].max(initial=0):.2e} "
                      f"worst dlin(ln<-5) {dlin[~hi].max(initial=0):.2e} bad {int(bad.sum())}/{bad.size}")
                if tag == 'gpu' and bad.any():
                    for o in np.argsort(-(np.where(hi, dln / 1e-3, dlin / 1e-4)).ravel())[:3]:
                        v, i = divmod(int(o), c['m'])
                        print(f"    v {v} bit {i}: gpu {g[v, i]:.6f} oracle {soft[v, i]:.6f} twin {soft32[v, i]:.6f}")
