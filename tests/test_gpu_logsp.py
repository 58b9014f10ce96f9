"""GPU parity of the conventional Log-SP decoder (NBLDPC_ALG_LOG_SP; SURVEY 8(f)
row 2) against the oracle's O-LS.

Bar (as for the Log-Fourier path): symbol-MAP hard decisions, syndrome flags
and iteration counts bit-exact on every stable frame (O-LS's fp64 and fp32 trajectories agree);
unstable frames are counted and must stay rare."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle
import synth
from helpers import DEFAULT_POLY
from parity import assert_stable_parity, config_inputs, oracle_code

pytestmark = pytest.mark.gpu

ALG_LOG_SP = 1


@pytest.fixture(scope="module")
def dev():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch.device("cuda:0")


def _compare(ocode, out, x, idx, max_iters, pmf=False):
    """Bit-exact on stable frames (assert_stable_parity, with O-LS's fp64 / fp32 runs); returns the number
    of unstable differing frames among idx."""
    ref = ocode.ls_decode_batch(x[idx], max_iters, pmf=pmf)
    got = {k: out[k].cpu().numpy()[idx] for k in ("hard", "ok", "iters")}
    return assert_stable_parity(ocode.ls_decode_batch, x[idx], got, ref, max_iters, max_unstable_frac=1.0,
                                what="Log-SP", pmf=pmf)


def _gpu(name):
    import paper_1008_4370_b200 as nb

    c = synth.CONFIGS[name]
    M, rows, cols, coeffs = synth.config_code(name)
    return nb.Code(c["m"], c["poly"], M, c["N"], rows, cols, coeffs)


@pytest.mark.parametrize("name,point,F,nsample", [("C1", 0, 64, 64), ("C2", 0, 64, 4), ("C5", 4, 64, 4)])
def test_logsp_decode_parity(dev, name, point, F, nsample):
    c = synth.CONFIGS[name]
    _, llr, _ = config_inputs(name, 0, F, point=point)
    code = _gpu(name)
    out = code.decode(torch.from_numpy(llr).to(dev), c["max_iters"], algorithm=ALG_LOG_SP)
    torch.cuda.synchronize()
    idx = np.arange(F) if nsample >= F else np.sort(np.random.default_rng(5).choice(F, nsample, replace=False))
    ocode = oracle_code(name)
    assert _compare(ocode, out, llr, idx, c["max_iters"]) <= max(1, len(idx) // 10)
    hard, okg = out["hard"].cpu().numpy(), out["ok"].cpu().numpy()
    for f in range(0, F, 4):
        assert bool(okg[f]) == ocode.syndrome(hard[f])[0]
    # the same frames in another batch and a repeat give identical results
    again = code.decode(torch.from_numpy(llr[::-1].copy()).to(dev), c["max_iters"], algorithm=ALG_LOG_SP)
    for k in ("hard", "ok", "iters"):
        assert torch.equal(again[k].flip(0), out[k]), k


def test_logsp_large_field_and_irregular(dev):
    import paper_1008_4370_b200 as nb

    # GF(256) (the q^2 check node at its largest) and GF(8) with check degrees 2..6
    for m, N, k, seed in [(8, 48, 4, 91), (3, 40, None, 92)]:
        if k is None:
            degs = [2, 3, 4, 5, 6] + [4] * 15  # sum = 80 = 2N
            from test_gpu_parity import _irregular_code
            M, rows, cols, coeffs = _irregular_code(N, degs, m, seed)
        else:
            M, rows, cols, coeffs = synth.make_regular_code(N, k, m, seed)
        code = nb.Code(m, DEFAULT_POLY[m], M, N, rows, cols, coeffs)
        ocode = oracle.Code(oracle.Field(m, DEFAULT_POLY[m]), M, N, rows, cols, coeffs)
        llr = synth.awgn_llr(N * m, 0, 16, synth.sigma2_for(2.0, 0.5), 300 + m)
        out = code.decode(torch.from_numpy(llr).to(dev), 20, algorithm=ALG_LOG_SP)
        assert _compare(ocode, out, llr, np.arange(16), 20) <= 2


def test_logsp_pmf_input(dev):
    name = "C1"
    c = synth.CONFIGS[name]
    _, _, xs = config_inputs(name, 0, 64)
    pmf = synth.config_pmf(name, 0, 64, ebn0_db=2.0, symbols=xs)
    code = _gpu(name)
    out = code.decode_pmf(torch.from_numpy(pmf).to(dev), c["max_iters"], algorithm=ALG_LOG_SP)
    assert _compare(oracle_code(name), out, pmf, np.arange(64), c["max_iters"], pmf=True) <= 6


def test_logsp_options_and_errors(dev):
    import paper_1008_4370_b200 as nb

    name = "C1"
    c = synth.CONFIGS[name]
    _, llr, _ = config_inputs(name, 0, 8)
    code = _gpu(name)
    x = torch.from_numpy(llr).to(dev)
    for kw in (dict(want_soft=True), dict(want_events=True), dict(want_post=True), dict(syndrome_mode=1)):
        with pytest.raises(nb.NbldpcError) as ei:
            code.decode(x, 10, algorithm=ALG_LOG_SP, **kw)
        assert ei.value.status == -1
    with pytest.raises(nb.NbldpcError):
        code.decode(x, 10, algorithm=7)
    # max_iters = 1 and no early stop
    o = code.decode(x, 1, algorithm=ALG_LOG_SP)
    assert (o["iters"] == 1).all()
    o = code.decode(x, 5, algorithm=ALG_LOG_SP, early_stop=False)
    assert (o["iters"] == 5).all()
    ocode = oracle_code(name)
    ref = ocode.ls_decode_batch(llr, 5, early_stop=False)
    assert_stable_parity(ocode.ls_decode_batch, llr, {k: v.cpu().numpy() for k, v in o.items()}, ref, 5,
                         max_unstable_frac=0.25, what="Log-SP, 5 iterations, no early stop", early_stop=False)
    # end to end with host buffers
    h = code.decode_host(torch.from_numpy(llr).pin_memory(), c["max_iters"], algorithm=ALG_LOG_SP)
    d = code.decode(x, c["max_iters"], algorithm=ALG_LOG_SP)
    for k in ("hard", "ok", "iters"):
        assert torch.equal(d[k].cpu(), h[k])
