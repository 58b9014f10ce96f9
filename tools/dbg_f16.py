"""FER / undetected-error / iteration comparison of F32 and F16 messages (diagnostic)."""
import sys

import numpy as np
import torch

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import synth  # noqa: E402
from parity import config_inputs  # noqa: E402

import paper_1008_4370_b200 as nb  # noqa: E402

for name, point, F in [("C2", 0, 4096), ("C3", 0, 2048), ("C4", 0, 256), ("C5", 0, 4096), ("C5", 3, 8192)]:
    c = synth.CONFIGS[name]
    _, llr, xs = config_inputs(name, 0, F, point=point)
    M, rows, cols, coeffs = synth.config_code(name)
    code = nb.Code(c["m"], c["poly"], M, c["N"], rows, cols, coeffs)
    x = torch.from_numpy(llr).cuda()
    res = []
    for fmt in (0, 1):
        o = code.decode(x, c["max_iters"], message_format=fmt)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); o = code.decode(x, c["max_iters"], message_format=fmt); e1.record(); torch.cuda.synchronize()
        ok = o["ok"].cpu().numpy().astype(bool)
        hard = o["hard"].cpu().numpy()
        wrong = ~(hard == xs.astype(np.uint8)).all(1)
        it = o["iters"].cpu().numpy()
        res.append((fmt, 1 - ok.mean(), (ok & wrong).mean(), it.mean(), e0.elapsed_time(e1) * 1e6 / it.sum()))
    print(name, point, " | ".join("fmt%d FER %.4f undet %.4f iters %.2f ns/fi %.0f" % r for r in res))
