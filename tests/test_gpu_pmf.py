"""GPU parity of the symbol-pmf input (nbldpc_decode_pmf) against the oracle.

Inputs: q-ary orthogonal signalling over AWGN (synth.orthogonal_pmf), a channel whose pmf does
not factor over the bits.  Same bar as the LLR path: hard decisions,
syndrome flags and iteration counts bit-exact on every stable frame (fp64 and fp32 oracle
trajectories agree); per step (nbldpc_step_pmf, from the oracle's state) messages within 1e-3 ln /
1e-4 linear and soft outputs under the north-star bar."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import synth
from helpers import bit_prior
from parity import assert_stable_parity, config_inputs, oracle_code, soft_mismatch

pytestmark = pytest.mark.gpu

_codes = {}


def gpu_code(name):
    import paper_1008_4370_b200 as nb

    if name not in _codes:
        c = synth.CONFIGS[name]
        M, rows, cols, coeffs = synth.config_code(name)
        _codes[name] = nb.Code(c["m"], c["poly"], M, c["N"], rows, cols, coeffs)
    return _codes[name]


@pytest.fixture(scope="module")
def dev():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch.device("cuda:0")


def _pmf_inputs(name, F, ebn0):
    _, _, xs = config_inputs(name, 0, F)
    return synth.config_pmf(name, 0, F, ebn0_db=ebn0, symbols=xs), xs


def _compare(name, out, pmf, idx, max_iters):
    """Bit-exact on stable frames (assert_stable_parity); returns the number of unstable frames among idx."""
    ocode = oracle_code(name)
    ref = ocode.lf_decode_batch_pmf(pmf[idx], max_iters)
    got = {k: out[k].cpu().numpy()[idx] for k in ("hard", "ok", "iters")}
    return assert_stable_parity(ocode.lf_decode_batch_pmf, pmf[idx], got, ref, max_iters, what=name)


PMF_CASES = [
    # name, Eb/N0 (dB), gpu frames, oracle sample
    ("C1", 2.0, 64, 64),
    ("C2", 0.5, 256, 8),
    ("C3", 1.0, 64, 4),
    ("C5", 3.5, 256, 16),
]


@pytest.mark.parametrize("vn", [0, 1])
@pytest.mark.parametrize("name,ebn0,F,nsample", PMF_CASES)
def test_pmf_decode_parity(dev, name, ebn0, F, nsample, vn):
    # vn 0: the cluster kernel's pmf variant (default); 1: the slot-pass kernel's
    c = synth.CONFIGS[name]
    pmf, xs = _pmf_inputs(name, F, ebn0)
    code = gpu_code(name)
    out = code.decode_pmf(torch.from_numpy(pmf).to(dev), c["max_iters"], vn_algorithm=vn)
    torch.cuda.synchronize()
    rng = np.random.default_rng(2)
    idx = np.arange(F) if nsample >= F else np.sort(rng.choice(F, nsample, replace=False))
    unstable = _compare(name, out, pmf, idx, c["max_iters"])
    assert unstable <= max(1, len(idx) // 10)
    it = out["iters"].cpu().numpy()
    assert it.min() >= 1 and it.max() <= c["max_iters"]
    ocode = oracle_code(name)
    hard, okg = out["hard"].cpu().numpy(), out["ok"].cpu().numpy()
    for f in rng.choice(F, min(F, 32), replace=False):
        assert bool(okg[f]) == ocode.syndrome(hard[f])[0]


@pytest.mark.parametrize("vn", [0, 1])
@pytest.mark.parametrize("name", ["C1"])
def test_pmf_soft_parity(dev, name, vn):
    # posterior bit log-magnitudes of a one-iteration decode: the north-star bar (1e-3 ln where ln >= -5,
    # else 1e-4 linear).  A decode's soft output also carries the fp32 first check-node step (P^0 = WHT(p)
    # and W^(1) in fp32), so the bar on the decision itself is checked per step from the oracle's own
    # state, for C1, C5, C2 and C3 in test_pmf_step_parity.
    pmf, _ = _pmf_inputs(name, 64 if name == "C1" else 16, 2.0 if name == "C1" else 3.5)
    code = gpu_code(name)
    ocode = oracle_code(name)
    out = code.decode_pmf(torch.from_numpy(pmf).to(dev), 1, early_stop=False, want_soft=True, want_events=True,
                          vn_algorithm=vn)
    ref = ocode.lf_decode_batch_pmf(pmf, 1, early_stop=False, want_soft=True)
    soft = out["soft"].cpu().numpy()
    bad = soft_mismatch(soft, ref["soft"])
    assert not bad.any(), (int(bad.sum()), float(np.abs(soft - ref["soft"])[bad].max(initial=0)))
    assert int(out["events"].sum()) == 0


@pytest.mark.parametrize("name,ell,F", [("C1", 1, 4), ("C1", 3, 4), ("C5", 1, 2), ("C5", 2, 2), ("C5", 3, 2),
                                        ("C2", 2, 2), ("C2", 3, 2), ("C3", 2, 2), ("C3", 3, 2)])
def test_pmf_step_parity(dev, name, ell, F):
    """One Log-Fourier iteration with the symbol-pmf channel (nbldpc_step_pmf) from the oracle's state
    W^(ell) (O-LF with lf_init_pmf), rounded to the packed f32 format: U within 1e-3 ln / 1e-4 linear; W
    within (k-1) 1e-3; the check node on the GPU's own U within (k-1) 1e-3; soft outputs under the
    north-star bar; hard decisions equal away from ties -- for the soft-output (packed log) and the
    hot-path (linear messages at q >= 128) instantiations."""
    from parity import message_mismatch, oracle_to_packed, packed_to_oracle

    c = synth.CONFIGS[name]
    pmf, _ = _pmf_inputs(name, F, {"C1": 2.0, "C5": 3.5, "C2": 0.5, "C3": 1.0}[name])
    ocode = oracle_code(name)
    code = gpu_code(name)
    ecol = ocode.edges()[1]
    w_in, refs = [], []
    for f in range(F):
        S0, L0 = ocode.lf_init_pmf(pmf[f].astype(np.float64))
        Us, Ul = S0[ecol].copy(), L0[ecol].copy()
        for _ in range(ell):
            Ws, Wl = ocode.lf_check_to_variable(Us, Ul)
            Us, Ul, _ = ocode.lf_variable_to_check(S0, L0, Ws, Wl)
        packed = oracle_to_packed(Ws, Wl)
        w_in.append(packed)
        Ws32, Wl32 = packed_to_oracle(packed)
        Us, Ul, _ = ocode.lf_variable_to_check(S0, L0, Ws32, Wl32)
        x, soft, _ = ocode.lf_decision(S0, L0, Ws32, Wl32)
        Wn_s, Wn_l = ocode.lf_check_to_variable(Us, Ul)
        refs.append((Us, Ul, x, soft, Wn_s, Wn_l))
    w_in = torch.from_numpy(np.stack(w_in)).to(dev)
    p = torch.from_numpy(pmf).to(dev)
    runs = [(True, code.step_pmf(p, ell, w_in, want_u=True, want_soft=True)),
            (False, code.step_pmf(p, ell, w_in, want_u=True, want_soft=False))]
    torch.cuda.synchronize()
    k1 = c["k"] - 1
    for soft_run, res in runs:
        for f in range(F):
            Us, Ul, x, soft, Wn_s, Wn_l = refs[f]
            what = f"{name} l={ell} {'soft' if soft_run else 'plain'} kernel, frame {f}"
            gus, gul = packed_to_oracle(res["u"][f].cpu().numpy())
            assert message_mismatch(gus, gul, Us, Ul).sum() == 0, what + ": U"
            gs, gl = packed_to_oracle(res["w"][f].cpu().numpy())
            cn_s, cn_l = ocode.lf_check_to_variable(gus, gul)
            assert message_mismatch(gs, gl, cn_s, cn_l, ln_tol=1e-3 * k1).sum() == 0, what + ": check node"
            assert message_mismatch(gs, gl, Wn_s, Wn_l, ln_tol=1e-3 * k1).sum() == 0, what + ": W"
            hard = res["hard"][f].cpu().numpy()
            sure = (soft > -12.0).all(1)
            assert np.array_equal(hard[sure], x[sure]), what + ": hard"
            if soft_run:
                gsoft = res["soft"][f].cpu().numpy().reshape(c["N"], c["m"])
                bad = soft_mismatch(gsoft, soft)
                assert not bad.any(), (what, int(bad.sum()), float(np.abs(gsoft - soft)[bad].max(initial=0)))


@pytest.mark.parametrize("vn", [0, 1])
def test_factorised_pmf_equals_llr_path(dev, vn):
    # a bit-product pmf is the LLR input in another form: same decisions
    name = "C5"
    c = synth.CONFIGS[name]
    _, llr, _ = config_inputs(name, 0, 128, point=4)
    m, N = c["m"], c["N"]
    pmf = np.stack([np.stack([bit_prior(f[v * m:(v + 1) * m].astype(np.float64)) for v in range(N)])
                    for f in llr]).astype(np.float32)
    code = gpu_code(name)
    a = code.decode(torch.from_numpy(llr).to(dev), c["max_iters"], vn_algorithm=vn)
    b = code.decode_pmf(torch.from_numpy(pmf).to(dev), c["max_iters"], vn_algorithm=vn)
    same = ((a["hard"] == b["hard"]).all(1) & (a["ok"] == b["ok"]) & (a["iters"] == b["iters"])).float().mean()
    assert same.item() >= 0.95


def test_pmf_invariance_and_edge_cases(dev):
    import paper_1008_4370_b200 as nb

    name = "C2"
    c = synth.CONFIGS[name]
    pmf, _ = _pmf_inputs(name, 96, 0.5)
    code = gpu_code(name)
    x = torch.from_numpy(pmf).to(dev)
    base = code.decode_pmf(x, c["max_iters"])
    base1 = code.decode_pmf(x, c["max_iters"], vn_algorithm=1)
    for kw in (dict(slots=1), dict(slots=13), dict(vn_algorithm=1, slots=7), dict(vn_algorithm=1, use_graph=-1, slots=5)):
        o = code.decode_pmf(x, c["max_iters"], **kw)
        ref = base1 if kw.get("vn_algorithm") else base
        for k in ("hard", "ok", "iters"):
            assert torch.equal(o[k], ref[k]), (kw, k)
    # row scale does not matter (rows are scaled to probabilities, reading R23)
    o = code.decode_pmf(x * 3.5, c["max_iters"])
    same = ((o["hard"] == base["hard"]).all(1) & (o["iters"] == base["iters"])).float().mean()
    assert same.item() >= 0.95
    # the LLR path on the same handle is unaffected by a pmf decode in between
    _, llr, _ = config_inputs(name, 0, 32)
    l1 = code.decode(torch.from_numpy(llr).to(dev), c["max_iters"])
    code.decode_pmf(x, c["max_iters"])
    l2 = code.decode(torch.from_numpy(llr).to(dev), c["max_iters"])
    for k in ("hard", "ok", "iters"):
        assert torch.equal(l1[k], l2[k])
    # point masses on the sent (all-zero) codeword: converged at the first iteration
    pm = torch.zeros_like(x[:4])
    pm[..., 0] = 1.0
    o = code.decode_pmf(pm.contiguous(), c["max_iters"], want_events=True)
    assert (o["iters"] == 1).all() and (o["ok"] == 1).all() and not o["hard"].any()
    # a row with zero sum is treated as uniform and counted as an event
    z = x[:2].clone()
    z[0, 5] = 0.0
    for vn in (0, 1):
        o = code.decode_pmf(z, c["max_iters"], want_events=True, vn_algorithm=vn)
        assert int(o["events"][0]) >= 1 and int(o["events"][1]) == 0
    # argument errors
    with pytest.raises(ValueError):
        code.decode_pmf(x[:, :, :-1].contiguous(), 10)
    flat = torch.zeros(x[:1].numel() + 1, device=dev)
    L = nb.lib()
    h = torch.zeros((1, c["N"]), dtype=torch.uint8, device=dev)
    k = torch.zeros(1, dtype=torch.uint8, device=dev)
    i = torch.zeros(1, dtype=torch.int32, device=dev)
    st = L.nbldpc_decode_pmf(code._h, flat.data_ptr() + 4, 1, 10, h.data_ptr(), k.data_ptr(), i.data_ptr(),
                             None, None)
    assert st == -1  # misaligned pmf


POST_CASES = [
    # name, input, Eb/N0 or LLR point, gpu frames, oracle sample
    ("C1", "llr", 0, 64, 32),
    ("C5", "pmf", 3.5, 128, 8),
    ("C2", "pmf", 0.5, 64, 4),
    ("C3", "llr", 0, 32, 3),
    ("C2", "llr", 0, 64, 4),  # the q = 64 symbol-output variant of the cluster kernel (no work rows)
]


@pytest.mark.parametrize("vn", [0, 1])
@pytest.mark.parametrize("name,kind,pt,F,nsample", POST_CASES)
def test_symbol_posterior_and_map_parity(dev, name, kind, pt, F, nsample, vn):
    # LLR input: vn 0 the cluster kernel's symbol-output variant, vn 1 the slot-pass kernel;
    # pmf input: the pass kernel either way
    # symbol-level TENTATIVE DECISION at the stopping iteration (reading R24):
    # per frame the posterior is within 1e-4 of the fp64 oracle or no further than twice the
    # oracle's own fp32 twin (the message state carries fp32 rounding into an uncertain posterior),
    # over the sample no further than the twin in total; MAP equal where the top two are apart
    c = synth.CONFIGS[name]
    code = gpu_code(name)
    ocode = oracle_code(name)
    if kind == "pmf":
        x, _ = _pmf_inputs(name, F, pt)
        out = code.decode_pmf(torch.from_numpy(x).to(dev), c["max_iters"], want_post=True)
        plain = code.decode_pmf(torch.from_numpy(x).to(dev), c["max_iters"], vn_algorithm=1)
    else:
        _, x, _ = config_inputs(name, 0, F, point=pt)
        out = code.decode(torch.from_numpy(x).to(dev), c["max_iters"], want_post=True, vn_algorithm=vn)
        plain = code.decode(torch.from_numpy(x).to(dev), c["max_iters"], vn_algorithm=vn)
    for k in ("hard", "ok", "iters"):  # the symbol outputs do not perturb the decode
        assert torch.equal(out[k], plain[k]), k
    idx = np.sort(np.random.default_rng(3).choice(F, nsample, replace=False))
    dec = ocode.lf_decode_batch_pmf if kind == "pmf" else ocode.lf_decode_batch
    ref = dec(x[idx], c["max_iters"], want_post=True)
    twin = dec(x[idx], c["max_iters"], want_post=True, f32=True)
    post = out["post"].cpu().numpy()[idx]
    xmap = out["map"].cpu().numpy()[idx]
    it = out["iters"].cpu().numpy()[idx]
    checked, eg_tot, et_tot = 0, 0.0, 0.0
    for n in range(len(idx)):
        stable = np.array_equal(twin["hard"][n], ref["hard"][n]) and twin["iters"][n] == ref["iters"][n]
        if not stable or it[n] != ref["iters"][n]:
            continue
        checked += 1
        np.testing.assert_allclose(post[n].sum(1), 1.0, atol=1e-4)
        eg = np.abs(post[n] - ref["post"][n]).max()
        et = np.abs(twin["post"][n] - ref["post"][n]).max()
        assert eg <= max(1e-4, 2.0 * et), (n, eg, et)
        eg_tot, et_tot = eg_tot + eg, et_tot + et
        top2 = np.sort(ref["post"][n], 1)[:, -2:]
        clear = top2[:, 1] - top2[:, 0] > 2.0 * max(1e-4, 2.0 * et)
        assert np.array_equal(xmap[n][clear], ref["map"][n][clear])
    assert checked >= max(1, (len(idx) * 3) // 4)
    assert eg_tot <= max(1e-4 * checked, 1.25 * et_tot)


def test_pmf_host_entry_matches_device(dev):
    # nbldpc_decode_pmf_host (chunked copy overlapped with the decode) = the device entry
    name = "C2"
    c = synth.CONFIGS[name]
    pmf, _ = _pmf_inputs(name, 640, 0.5)
    code = gpu_code(name)
    d = code.decode_pmf(torch.from_numpy(pmf).to(dev), c["max_iters"])
    for vn in (0, 1):
        h = code.decode_pmf_host(torch.from_numpy(pmf).pin_memory(), c["max_iters"], vn_algorithm=vn)
        ref = d if vn == 0 else code.decode_pmf(torch.from_numpy(pmf).to(dev), c["max_iters"], vn_algorithm=1)
        for k in ("hard", "ok", "iters"):
            assert torch.equal(ref[k].cpu(), h[k]), (vn, k)
