"""Debug aid: per-step soft output of the GPU vs the oracle (C3, l = 3) and the worst entries."""
import sys
import numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import synth, paper_1008_4370_b200 as nb
from parity import config_inputs, oracle_code, oracle_to_packed, packed_to_oracle
name, ell = sys.argv[1], int(sys.argv[2])
c = synth.CONFIGS[name]; F = 2
_, llr, _ = config_inputs(name, 0, F)
oc = oracle_code(name); M, rows, cols, coeffs = synth.config_code(name)
code = nb.Code(c['m'], c['poly'], M, c['N'], rows, cols, coeffs)
ecol = oc.edges()[1]
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
    refs.append((soft, soft32))
res = code.step(torch.from_numpy(llr).cuda(), ell, torch.from_numpy(np.stack(w_in)).cuda(), want_soft=True)
torch.cuda.synchronize()
for f in range(F):
    soft, soft32 = refs[f]
    g = res['soft'][f].cpu().numpy().reshape(c['N'], c['m'])
    dln = np.abs(g - soft); dlin = np.abs(np.exp(g.astype(np.float64)) - np.exp(soft))
    bad = (dln > np.maximum(1e-3, np.abs(soft32 - soft))) & (dlin > 1e-4)
    order = np.argsort(-dln.ravel())[:6]
    for o in order:
        v, i = divmod(int(o), c['m'])
        print(f, 'v', v, 'bit', i, 'gpu %.6f oracle %.6f twin %.6f dln %.2e dlin %.2e bad %d' % (g[v, i], soft[v, i], soft32[v, i], dln[v, i], dlin[v, i], bad[v, i]))
