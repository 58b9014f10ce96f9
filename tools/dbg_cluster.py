"""Debug aid: small decodes on the cluster kernel vs the oracle."""
import sys
import numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import synth, paper_1008_4370_b200 as nb
from parity import config_inputs, oracle_code
for name, F, slots, mi in [("C1", 4, 1, 1), ("C1", 4, 1, 20), ("C1", 4, 2, 20), ("C1", 64, 0, 20), ("C2", 8, 1, 50), ("C2", 8, 0, 50)]:
    c = synth.CONFIGS[name]
    M, rows, cols, coeffs = synth.config_code(name)
    code = nb.Code(c['m'], c['poly'], M, c['N'], rows, cols, coeffs)
    _, llr, _ = config_inputs(name, 0, F)
    out = code.decode(torch.from_numpy(llr).cuda(), mi, slots=slots)
    torch.cuda.synchronize()
    ref = oracle_code(name).lf_decode_batch(llr, mi)
    it = out['iters'].cpu().numpy(); ok = out['ok'].cpu().numpy(); h = out['hard'].cpu().numpy()
    print(name, F, slots, mi, 'gpu iters', it[:8], 'ref', ref['iters'][:8], 'ok', ok[:8], ref['ok'][:8],
          'hard eq', (h == ref['hard']).all(1)[:8], flush=True)
