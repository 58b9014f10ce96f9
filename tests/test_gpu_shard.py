"""The N>1 path with real GPU decodes: two ranks (gloo process group, both on
cuda:0 -- the pool has one GPU per call; the ranks' kernels never wait on one another, the only
collectives come after decoding) each decode their strong-scaling shard of a fixed global batch
through the C-ABI.  The all-gathered outputs and the all-reduced counter vector must be identical to
one single-process decode of the whole batch."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import synth

pytestmark = pytest.mark.gpu

CASES = [("C4", 0, 512), ("C5", 3, 1024)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _decode(name, point, f0, n):
    import paper_1008_4370_b200 as nb

    c = synth.CONFIGS[name]
    M, rows, cols, coeffs = synth.config_code(name)
    code = nb.Code(c["m"], c["poly"], M, c["N"], rows, cols, coeffs)
    llr = torch.from_numpy(synth.config_llr(name, f0, n, point=point)).cuda()
    out = code.decode(llr, c["max_iters"], want_events=True)
    torch.cuda.synchronize()
    return out


def _counts(out):
    from paper_1008_4370_b200 import shard

    c = shard.error_counts(out["hard"], out["ok"], None, out["events"])
    c["frame_iters"] = int(out["iters"].to(torch.int64).sum().item())
    return c


def _worker(rank, world, port, name, point, F, q):
    import torch.distributed as dist

    from paper_1008_4370_b200 import shard

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, b = shard.frame_range(rank, world, F, "strong")
        out = _decode(name, point, a, b - a)
        c, _ = shard.reduce_stats(_counts(out), {"ms": 1.0}, dist)
        sizes = [(lambda x, y: y - x)(*shard.frame_range(g, world, F, "strong")) for g in range(world)]
        g = {k: shard.gather_rows(out[k].cpu(), dist, sizes).numpy() for k in ("hard", "ok", "iters", "events")}
        q.put((rank, c, g))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,point,F", CASES)
def test_strong_scaling_shards_equal_single_process(name, point, F):
    import torch.multiprocessing as mp

    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, point, F, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    whole = _decode(name, point, 0, F)
    want = _counts(whole)
    for _, c, g in res:
        assert c == want, (c, want)
        for k in ("hard", "ok", "iters", "events"):
            assert np.array_equal(g[k], whole[k].cpu().numpy()), k
