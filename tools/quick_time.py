"""Quick timing of decode on one config (development aid, not the bench contract)."""
import sys, time, json
import numpy as np, torch
sys.path.insert(0, '.')
import synth, paper_1008_4370_b200 as nb
name = sys.argv[1] if len(sys.argv) > 1 else 'C2'
F = int(sys.argv[2]) if len(sys.argv) > 2 else synth.CONFIGS[name]['frames']
slots = int(sys.argv[3]) if len(sys.argv) > 3 else 0
point = int(sys.argv[4]) if len(sys.argv) > 4 else 0
c = synth.CONFIGS[name]
M, r, co, h = synth.config_code(name)
code = nb.Code(c['m'], c['poly'], M, c['N'], r, co, h)
llr = torch.from_numpy(synth.config_llr(name, 0, F, point=point)).cuda()
for g in (0, -1):
    out = code.decode(llr, c['max_iters'], slots=slots, use_graph=g); torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); out = code.decode(llr, c['max_iters'], slots=slots, use_graph=g); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    it = out['iters'].cpu().numpy(); ok = out['ok'].cpu().numpy()
    K = c['N'] * c['m'] * c['rate']
    t = min(ts) * 1e-3
    fma = it.sum() * (2 * c['N'] * c['q'] ** 2 + c['N'] * (c['m'] + 1) * c['q'])
    print(json.dumps(dict(cfg=name, F=F, graph=g, slots=slots, ms=min(ts), mean_iters=float(it.mean()), max_iters=int(it.max()),
          ok=float(ok.mean()), metric=float(K * it.sum() / t), tflops=float(2 * fma / t / 1e12), frac_fma=float(fma / t / 37.2e12))))
