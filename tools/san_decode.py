"""Small decodes for compute-sanitizer runs (C1 all frames, C2 / C5 / C3 a few frames, both VN algorithms)."""
import sys
import torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import synth, paper_1008_4370_b200 as nb
from parity import config_inputs
for name, F, mi in [("C1", 64, 20), ("C2", 6, 6), ("C5", 4, 4), ("C3", 3, 3)]:
    c = synth.CONFIGS[name]
    M, rows, cols, coeffs = synth.config_code(name)
    code = nb.Code(c['m'], c['poly'], M, c['N'], rows, cols, coeffs)
    _, llr, _ = config_inputs(name, 0, F)
    x = torch.from_numpy(llr).cuda()
    for vn in (0, 1):
        out = code.decode(x, mi, vn_algorithm=vn, want_soft=True)
        torch.cuda.synchronize()
        print(name, vn, out['iters'].tolist()[:6], flush=True)
