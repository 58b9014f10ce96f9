"""Quick timing of decode on one config (development aid, not the bench contract).
usage: python tools/quick_time.py CFG [frames] [slots] [point] [vn list e.g. 0,1] [graph list e.g. 0,-1]"""
import os, sys, json
import torch
sys.path.insert(0, '.')
import synth, paper_1008_4370_b200 as nb
name = sys.argv[1] if len(sys.argv) > 1 else 'C2'
F = int(sys.argv[2]) if len(sys.argv) > 2 and int(sys.argv[2]) > 0 else synth.CONFIGS[name]['frames']
slots = int(sys.argv[3]) if len(sys.argv) > 3 else 0
point = int(sys.argv[4]) if len(sys.argv) > 4 else 0
vns = [int(x) for x in sys.argv[5].split(',')] if len(sys.argv) > 5 else [0]
graphs = [int(x) for x in sys.argv[6].split(',')] if len(sys.argv) > 6 else [0]
c = synth.CONFIGS[name]
M, r, co, h = synth.config_code(name)
code = nb.Code(c['m'], c['poly'], M, c['N'], r, co, h)
llr = torch.from_numpy(synth.config_llr(name, 0, F, point=point)).cuda()
for vn in vns:
    for g in graphs:
        es = not os.environ.get('NO_EARLY')
        mf = int(os.environ.get('MSG', '0'))  # 1: half-precision messages
        out = code.decode(llr, c['max_iters'], slots=slots, use_graph=g, vn_algorithm=vn, early_stop=es, message_format=mf); torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(); out = code.decode(llr, c['max_iters'], slots=slots, use_graph=g, vn_algorithm=vn, early_stop=es, message_format=mf); e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        it = out['iters'].cpu().numpy(); ok = out['ok'].cpu().numpy()
        K = c['N'] * c['m'] * c['rate']
        t = min(ts) * 1e-3
        fi = it.sum()
        print(json.dumps(dict(cfg=name, point=point, F=F, vn=vn, graph=g, slots=slots, ms=round(min(ts), 3),
                              mean_iters=float(it.mean()), ok=float(ok.mean()), metric=float(K * fi / t),
                              ns_per_frame_iter=1e9 * t / fi, launches=code.last_decode_launches())))
