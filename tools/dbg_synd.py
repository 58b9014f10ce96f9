import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np, torch, synth, paper_1008_4370_b200 as nb
from parity import config_inputs, oracle_code
name='C1'; c=synth.CONFIGS[name]
M, rows, cols, coeffs = synth.config_code(name)
for variant in ['orig','h1']:
    h = coeffs if variant=='orig' else np.ones_like(coeffs)
    code = nb.Code(c['m'], c['poly'], M, c['N'], rows, cols, h)
    oc = oracle_code(c, M, rows, cols, h)
    _, llr, xs = config_inputs(name, 0, 64)
    for it in (1,2,3):
        o = code.decode(torch.from_numpy(llr).cuda(), it, early_stop=False)
        hard = o['hard'].cpu().numpy(); ok = o['ok'].cpu().numpy()
        osyn = np.array([oc.syndrome(hard[f])[0] for f in range(64)])
        print(variant, it, 'gpu ok', ok.sum(), 'oracle-syndrome ok of gpu hard', osyn.sum(), 'mismatch', (ok != osyn).sum())
