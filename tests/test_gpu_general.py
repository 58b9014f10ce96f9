"""GPU parity of the general-column-weight Log-Fourier kernel (NBLDPC_VN_GENERAL, lf_general.cuh;
SURVEY 8(f) row 3) against the oracle's O-LF, which handles any column weight.

Bar as for the (2,k) path: hard decisions, syndrome flags and iteration
counts bit-exact on stable frames; soft outputs under R22, the symbol posterior under R24."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle
import synth
from helpers import DEFAULT_POLY
from parity import assert_stable_parity, config_inputs, oracle_code, soft_mismatch

pytestmark = pytest.mark.gpu
VN_GENERAL = 2


@pytest.fixture(scope="module")
def dev():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch.device("cuda:0")


def _codes(m, M, N, rows, cols, coeffs):
    import paper_1008_4370_b200 as nb

    return (nb.Code(m, DEFAULT_POLY[m], M, N, rows, cols, coeffs),
            oracle.Code(oracle.Field(m, DEFAULT_POLY[m]), M, N, rows, cols, coeffs))


def _compare(ocode, out, x, idx, max_iters, pmf=False):
    """Bit-exact on stable frames (assert_stable_parity); returns the number of unstable differing frames."""
    dec = ocode.lf_decode_batch_pmf if pmf else ocode.lf_decode_batch
    ref = dec(x[idx], max_iters)
    got = {k: out[k].cpu().numpy()[idx] for k in ("hard", "ok", "iters")}
    return assert_stable_parity(dec, x[idx], got, ref, max_iters, max_unstable_frac=1.0, what="general")


@pytest.mark.parametrize("m,N,k,j,ebn0", [(3, 96, 6, 3, 2.5), (4, 120, 6, 3, 2.0), (6, 64, 8, 4, 3.0),
                                          (8, 48, 6, 3, 2.5), (1, 240, 6, 3, 3.0)])
def test_general_decode_parity(dev, m, N, k, j, ebn0):
    M, rows, cols, coeffs = synth.make_regular_code(N, k, m, 200 + m, j=j)
    code, ocode = _codes(m, M, N, rows, cols, coeffs)
    F = 48
    llr = synth.awgn_llr(N * m, 0, F, synth.sigma2_for(ebn0, 1 - j / k), 400 + m)
    out = code.decode(torch.from_numpy(llr).to(dev), 30)
    torch.cuda.synchronize()
    idx = np.arange(F) if m <= 4 else np.arange(0, F, 4)
    assert _compare(ocode, out, llr, idx, 30) <= max(1, len(idx) // 10)
    okg, hard = out["ok"].cpu().numpy(), out["hard"].cpu().numpy()
    assert okg.mean() > 0.5
    for f in range(F):
        assert bool(okg[f]) == ocode.syndrome(hard[f])[0]


@pytest.mark.parametrize("name,point,F,nsample", [("C1", 0, 64, 64), ("C2", 0, 256, 8), ("C5", 4, 128, 8)])
def test_general_kernel_on_weight2_codes(dev, name, point, F, nsample):
    # the (2,k) configs through NBLDPC_VN_GENERAL: the same oracle, the same bar
    c = synth.CONFIGS[name]
    _, llr, _ = config_inputs(name, 0, F, point=point)
    M, rows, cols, coeffs = synth.config_code(name)
    import paper_1008_4370_b200 as nb

    code = nb.Code(c["m"], c["poly"], M, c["N"], rows, cols, coeffs)
    out = code.decode(torch.from_numpy(llr).to(dev), c["max_iters"], vn_algorithm=VN_GENERAL)
    idx = np.arange(F) if nsample >= F else np.sort(np.random.default_rng(9).choice(F, nsample, replace=False))
    assert _compare(oracle_code(name), out, llr, idx, c["max_iters"]) <= max(1, len(idx) // 10)


def test_general_mixed_weights_soft_posterior_pmf(dev):
    # column weights 1, 2 and 3 in one code; soft outputs, symbol posterior, pmf input, events
    m, N, k = 4, 64, 4
    M, rows, cols, coeffs = synth.make_regular_code(N, k, m, 211)
    rng = np.random.default_rng(211)
    extra = rng.choice(N, 24, replace=False)
    rows = np.concatenate([rows, M + np.arange(24) // 4])
    cols = np.concatenate([cols, extra])
    coeffs = np.concatenate([coeffs, rng.integers(1, 16, 24)])
    lone = np.setdiff1d(np.arange(N), extra)[:4]
    keep = np.ones(len(rows), bool)
    for v in lone:
        keep[np.where(cols == v)[0][0]] = False
    rows, cols, coeffs = rows[keep], cols[keep], coeffs[keep]
    order = np.lexsort((cols, rows))
    rows, cols, coeffs = rows[order], cols[order], coeffs[order]
    assert set(np.bincount(cols, minlength=N).tolist()) == {1, 2, 3}
    code, ocode = _codes(m, M + 6, N, rows, cols, coeffs)
    F = 32
    llr = synth.awgn_llr(N * m, 0, F, synth.sigma2_for(2.5, 0.4), 500)
    x = torch.from_numpy(llr).to(dev)
    out = code.decode(x, 25)
    assert _compare(ocode, out, llr, np.arange(F), 25) <= 3
    # soft (R22) and the symbol posterior (R24) after a fixed number of iterations
    for iters in (1, 3):
        o = code.decode(x, iters, early_stop=False, want_soft=True, want_post=True, want_events=True)
        ref = ocode.lf_decode_batch(llr, iters, early_stop=False, want_soft=True, want_post=True)
        twin = ocode.lf_decode_batch(llr, iters, early_stop=False, want_soft=True, want_post=True, f32=True)
        soft = o["soft"].cpu().numpy()
        bad = soft_mismatch(soft, ref["soft"])  # the north-star bar (fp64 decision for soft outputs)
        assert not bad.any(), (iters, int(bad.sum()))
        post = o["post"].cpu().numpy()
        ep = np.abs(post - ref["post"]).max()
        etp = np.abs(twin["post"] - ref["post"]).max()
        assert ep <= max(1e-4, 2.0 * etp), (iters, ep, etp)
        assert int(o["events"].sum()) == 0
    # pmf input on the same code
    pmf = synth.orthogonal_pmf(N, m, 0, F, synth.sigma2_for(1.5, 0.4), 600)
    out = code.decode_pmf(torch.from_numpy(pmf).to(dev), 25)
    assert _compare(ocode, out, pmf, np.arange(F), 25, pmf=True) <= 3


def test_general_unsupported_modes(dev):
    import paper_1008_4370_b200 as nb

    m, N, k = 3, 24, 6
    M, rows, cols, coeffs = synth.make_regular_code(N, k, m, 231, j=3)
    code, _ = _codes(m, M, N, rows, cols, coeffs)
    x = torch.from_numpy(synth.awgn_llr(N * m, 0, 4, 0.5, 1)).to(dev)
    with pytest.raises(nb.NbldpcError) as ei:
        code.decode(x, 10, syndrome_mode=1)
    assert ei.value.status == -1
    with pytest.raises(nb.NbldpcError) as ei:
        code.decode(x, 10, algorithm=1)  # Log-SP's fused variable node is the degree-2 one
    assert ei.value.status == -3
    with pytest.raises(nb.NbldpcError) as ei:
        code.step(x, 0)
    assert ei.value.status == -3
    E = __import__("ctypes").c_int()
    nb.lib().nbldpc_code_info(code._h, None, None, None, __import__("ctypes").byref(E), None)
    assert E.value == len(rows)
