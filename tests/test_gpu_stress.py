"""Race stress in place of compute-sanitizer racecheck/synccheck (closed on the GPU pool): the cluster
kernel's mbarrier / bulk-copy / fence.proxy.async pipeline and its cluster barriers are exercised
across cluster sizes (NBLDPC_CLUSTER_SIZE 1, 2, 4), slot counts and pipeline depths (NB_NSTAGE 2, 3,
a separate build), 20 repeats each.  The decoder has no float atomics on the data path, so every
repeat must be bit-identical to the first run: a missed barrier or an early buffer reuse shows up as a
difference in hard symbols, flags, iterations or soft outputs."""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import synth

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = [("C2", 0, 512), ("C3", 0, 256), ("C5", 3, 1024)]
REPEATS = 20


def _inputs(name, point, F):
    return torch.from_numpy(synth.config_llr(name, 0, F, point=point)).cuda()


def _code(name, cs=None):
    import paper_1008_4370_b200 as nb

    c = synth.CONFIGS[name]
    M, rows, cols, coeffs = synth.config_code(name)
    old = os.environ.get("NBLDPC_CLUSTER_SIZE")
    if cs is not None:
        os.environ["NBLDPC_CLUSTER_SIZE"] = str(cs)
    try:
        return nb.Code(c["m"], c["poly"], M, c["N"], rows, cols, coeffs)
    finally:
        if old is None:
            os.environ.pop("NBLDPC_CLUSTER_SIZE", None)
        else:
            os.environ["NBLDPC_CLUSTER_SIZE"] = old


def _run(code, x, max_iters, **kw):
    o = code.decode(x, max_iters, want_events=True, **kw)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in o.items()}


@pytest.mark.parametrize("name,point,F", CASES)
def test_repeat_invariance_cluster_sizes_and_slots(name, point, F):
    c = synth.CONFIGS[name]
    x = _inputs(name, point, F)
    base = _run(_code(name), x, c["max_iters"])
    for cs in (1, 2, 4):
        code = _code(name, cs)
        for slots in (0, 37, 148):
            for rep in range(REPEATS if slots == 0 else 4):
                o = _run(code, x, c["max_iters"], slots=slots)
                for k in base:
                    assert np.array_equal(o[k], base[k]), (name, cs, slots, rep, k)
    # soft outputs (the SOFT instantiation) and half-precision messages repeat bit-identically too
    code = _code(name)
    for kw in (dict(want_soft=True), dict(message_format=1)):
        s0 = _run(code, x, c["max_iters"], **kw)
        for rep in range(5):
            s = _run(code, x, c["max_iters"], **kw)
            for k in s0:
                assert np.array_equal(s[k], s0[k]), (name, kw, rep, k)


def test_three_stage_pipeline_build():
    """A build with NB_NSTAGE=3 (two chunks in flight per group) decodes bit-identically to the default
    two-stage build, 20 times over."""
    import tempfile

    from paper_1008_4370_b200 import build as nbuild

    if not os.path.exists(nbuild.NVCC):
        pytest.skip("nvcc not available")
    tmp = tempfile.mkdtemp(prefix="nb_nstage3_")
    lib = os.path.join(tmp, "libnbldpc.so")
    env = dict(os.environ, NBLDPC_LIB=lib, NBLDPC_DEFS="-DNB_NSTAGE=3")
    r = subprocess.run([sys.executable, "-c", "import paper_1008_4370_b200.build as b; b.build(force=True)"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, r.stderr[-3000:]
    base = {}
    for name, point, F in CASES:
        base[name] = _run(_code(name), _inputs(name, point, F), synth.CONFIGS[name]["max_iters"])
    ref = os.path.join(tmp, "base.npz")
    np.savez(ref, **{f"{n}:{k}": v for n, d in base.items() for k, v in d.items()})
    script = f"""
import sys, numpy as np, torch
sys.path.insert(0, {ROOT!r}); sys.path.insert(0, {os.path.join(ROOT, 'tests')!r})
import test_gpu_stress as t, synth
base = np.load({ref!r})
for name, point, F in t.CASES:
    c = synth.CONFIGS[name]
    code = t._code(name)
    x = t._inputs(name, point, F)
    for rep in range({REPEATS}):
        o = t._run(code, x, c['max_iters'])
        for k, v in o.items():
            assert np.array_equal(v, base[name + ':' + k]), (name, rep, k)
print('nstage3 ok')
"""
    r = subprocess.run([sys.executable, "-c", script], cwd=ROOT, env=env, capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0 and "nstage3 ok" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
