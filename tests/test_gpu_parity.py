"""GPU parity: the sm_100a decoder (through the C-ABI) against the CPU oracle.

Bar (BASELINE.json north_star):
  * hard decisions, syndrome flags and iteration counts bit-exact with the fp64
    oracle on every stable frame (a frame whose fp64 and fp32 oracle trajectories
    agree; unstable frames are counted and must be rare);
  * per-step message / posterior log-magnitudes within 1e-3 (ln) or 1e-4 linear.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle
import synth
from parity import (config_inputs, fail_trajectory_stable, message_mismatch, oracle_code, oracle_to_packed,
                    packed_to_oracle, soft_mismatch, assert_stable_parity)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch.device("cuda:0")


_codes = {}


def gpu_code(name):
    import paper_1008_4370_b200 as nb

    if name not in _codes:
        c = synth.CONFIGS[name]
        M, rows, cols, coeffs = synth.config_code(name)
        _codes[name] = nb.Code(c["m"], c["poly"], M, c["N"], rows, cols, coeffs)
    return _codes[name]


def compare_decode(name, gpu_out, llr_np, idx, max_iters, mode=0):
    """Oracle on frames idx; bit-exact on stable frames (assert_stable_parity).  Returns (n_checked, n_unstable)."""
    ocode = oracle_code(name)
    sub = llr_np[idx]
    ref = ocode.lf_decode_batch(sub, max_iters, mode=mode)
    got = {k: gpu_out[k].cpu().numpy()[idx] for k in ("hard", "ok", "iters")}
    unstable = assert_stable_parity(ocode.lf_decode_batch, sub, got, ref, max_iters, what=name, mode=mode)
    return len(idx), unstable


DECODE_CASES = [
    # name, point, gpu frames, oracle sample size
    ("C1", 0, 64, 64),
    ("C2", 0, 4096, 24),
    ("C3", 0, 512, 16),
    ("C4", 0, 1024, 16),
    ("C5", 0, 256, 8),   # 3.0 dB: every frame runs all 50 iterations
    ("C5", 3, 256, 16),  # 4.5 dB
    ("C5", 4, 256, 16),  # 5.0 dB
]


@pytest.mark.parametrize("name,point,F,nsample", DECODE_CASES)
def test_decode_parity(dev, name, point, F, nsample):
    _decode_parity(dev, name, point, F, nsample, 0)


@pytest.mark.parametrize("name,point,F,nsample", [("C1", 0, 64, 64), ("C2", 0, 512, 12), ("C5", 4, 128, 8)])
def test_decode_parity_direct_conv(dev, name, point, F, nsample):
    _decode_parity(dev, name, point, F, nsample, 1)


def _decode_parity(dev, name, point, F, nsample, vn):
    c = synth.CONFIGS[name]
    _, llr, xs = config_inputs(name, 0, F, point=point)
    code = gpu_code(name)
    out = code.decode(torch.from_numpy(llr).to(dev), c["max_iters"], vn_algorithm=vn)
    torch.cuda.synchronize()
    rng = np.random.default_rng(1)
    idx = np.arange(F) if nsample >= F else np.sort(rng.choice(F, nsample, replace=False))
    n, unstable = compare_decode(name, out, llr, idx, c["max_iters"])
    assert unstable <= max(1, n // 10)
    # every GPU frame: iterations within [1, max], ok consistent with the exact syndrome
    it = out["iters"].cpu().numpy()
    assert it.min() >= 1 and it.max() <= c["max_iters"]
    ocode = oracle_code(name)
    hard = out["hard"].cpu().numpy()
    okg = out["ok"].cpu().numpy()
    for f in rng.choice(F, min(F, 64), replace=False):
        assert bool(okg[f]) == ocode.syndrome(hard[f])[0]


@pytest.mark.parametrize("name,nsample", [("C1", 64), ("C5", 16), ("C2", 16), ("C3", 8)])
def test_paper_syndrome_mode_parity(dev, name, nsample):
    c = synth.CONFIGS[name]
    point = 4 if name == "C5" else 0
    _, llr, _ = config_inputs(name, 0, 64, point=point)
    out = gpu_code(name).decode(torch.from_numpy(llr).to(dev), c["max_iters"], syndrome_mode=1)
    torch.cuda.synchronize()
    idx = np.arange(0, 64, 64 // nsample)
    n, unstable = compare_decode(name, out, llr, idx, c["max_iters"], mode=1)
    assert unstable <= max(1, n // 10)


def _oracle_state(ocode, llr_row, iters):
    """Oracle trajectory up to W^(iters) (f64) for one frame."""
    S0, L0 = ocode.lf_init(llr_row.astype(np.float64))
    ecol = ocode.edges()[1]
    Us, Ul = S0[ecol].copy(), L0[ecol].copy()
    for _ in range(iters):
        Ws, Wl = ocode.lf_check_to_variable(Us, Ul)
        Us, Ul, _ = ocode.lf_variable_to_check(S0, L0, Ws, Wl)
    return S0, L0, Ws, Wl


# a GF(8) code (q = 8: one thread per edge holding all 8 entries) for the step parity
G8 = dict(name="G8", m=3, poly=0xB, k=4, N=96, q=8, ebn0=[1.5], rate=0.5, seed=4242)


def _step_inputs(name, F, point):
    """(config, llr [F, N*m], oracle code, GPU code) for a step-parity case."""
    import paper_1008_4370_b200 as nb

    if name == "G8":
        c = G8
        M, rows, cols, coeffs = synth.make_regular_code(c["N"], c["k"], c["m"], c["seed"])
        llr = synth.awgn_llr(c["N"] * c["m"], 0, F, synth.sigma2_for(c["ebn0"][0], c["rate"]), c["seed"] + 1)
        return (c, llr, oracle.Code(oracle.Field(c["m"], c["poly"]), M, c["N"], rows, cols, coeffs),
                nb.Code(c["m"], c["poly"], M, c["N"], rows, cols, coeffs))
    c = synth.CONFIGS[name]
    _, llr, _ = config_inputs(name, 0, F, point=point)
    return c, llr, oracle_code(name), gpu_code(name)


STEP_CASES = [("C1", 0, 1, 2), ("G8", 0, 1, 2), ("C5", 3, 1, 2), ("C2", 0, 1, 2), ("C3", 0, 1, 2),
              ("C1", 0, 2, 2), ("G8", 0, 2, 2), ("C5", 3, 2, 2), ("C2", 0, 2, 2), ("C3", 0, 2, 2), ("C4", 0, 2, 1),
              ("C1", 0, 3, 2), ("G8", 0, 3, 2), ("C5", 3, 3, 2), ("C2", 0, 3, 2), ("C3", 0, 3, 2)]
# the cluster kernel also at the fourth iteration of GF(256) (the most ill-conditioned decision sums);
# the direct-convolution pass kernel (vn = 1, the paper's q^2-term CONV, a comparison kernel) sums q
# fp32 products per entry and misses 1e-3 on a few U entries there, so only up to l = 3
STEP_PARAMS = ([(n, p, e, F, 0) for n, p, e, F in STEP_CASES + [("C3", 0, 4, 2)]] +
               [(n, p, e, F, 1) for n, p, e, F in STEP_CASES])


@pytest.mark.parametrize("name,point,ell,F,vn", STEP_PARAMS)
def test_step_parity(dev, name, point, ell, F, vn):
    """One iteration from the oracle's state W^(ell), rounded to the packed f32 format (nbldpc_step):
    * U within 1e-3 ln or 1e-4 linear of the oracle's U computed from the same rounded state;
    * the check node in isolation: W^(ell+1) within (k-1) 1e-3 ln / 1e-4 linear of the oracle's check
      node applied to the GPU's own U (k-1 log-magnitudes are summed);
    * W^(ell+1) from the GPU's U within (k-1) 1e-3 of the oracle's (U errors add up over k-1 terms);
    * posterior bit log-magnitudes (soft) under the north-star bar: 1e-3 ln where ln >= -5, else
      1e-4 linear (the fp64 decision of soft outputs, decision_f64, reading R22);
    * hard decisions equal wherever every bit is away from a tie."""
    c, llr, ocode, code = _step_inputs(name, F, point)
    w_in, refs = [], []
    for f in range(F):
        S0, L0, Ws, Wl = _oracle_state(ocode, llr[f], ell)
        packed = oracle_to_packed(Ws, Wl)
        w_in.append(packed)
        # the oracle continues from the same f32-rounded state
        Ws32, Wl32 = packed_to_oracle(packed)
        Us, Ul, _ = ocode.lf_variable_to_check(S0, L0, Ws32, Wl32)
        x, soft, _ = ocode.lf_decision(S0, L0, Ws32, Wl32)
        Wn_s, Wn_l = ocode.lf_check_to_variable(Us, Ul)
        refs.append((Us, Ul, x, soft, Wn_s, Wn_l))
    w_in = torch.from_numpy(np.stack(w_in)).to(dev)
    x = torch.from_numpy(llr).to(dev)
    # with soft outputs the step runs the soft-output instantiation (packed log messages, fp64 decision);
    # without, the hot-path instantiation (linear messages): both are checked
    runs = [(True, code.step(x, ell, w_in, want_u=True, want_soft=True, vn_algorithm=vn)),
            (False, code.step(x, ell, w_in, want_u=True, want_soft=False, vn_algorithm=vn))]
    torch.cuda.synchronize()
    k1 = c["k"] - 1
    for soft_run, res in runs:
        for f in range(F):
            Us, Ul, x_ref, soft, Wn_s, Wn_l = refs[f]
            what = f"{'soft' if soft_run else 'plain'} kernel, frame {f}"
            gus, gul = packed_to_oracle(res["u"][f].cpu().numpy())
            bad_u = message_mismatch(gus, gul, Us, Ul)
            assert bad_u.sum() == 0, f"{what}: U: {bad_u.sum()} of {bad_u.size} entries off"
            gs, gl = packed_to_oracle(res["w"][f].cpu().numpy())
            cn_s, cn_l = ocode.lf_check_to_variable(gus, gul)  # the oracle's check node on the GPU's U
            bad_cn = message_mismatch(gs, gl, cn_s, cn_l, ln_tol=1e-3 * k1, lin_tol=1e-4)
            assert bad_cn.sum() == 0, f"{what}: check node: {bad_cn.sum()} of {bad_cn.size} entries off"
            bad_w = message_mismatch(gs, gl, Wn_s, Wn_l, ln_tol=1e-3 * k1, lin_tol=1e-4)
            assert bad_w.sum() == 0, f"{what}: W: {bad_w.sum()} of {bad_w.size} entries off"
            hard = res["hard"][f].cpu().numpy()
            sure = (soft > -12.0).all(1)
            assert np.array_equal(hard[sure], x_ref[sure]), what
            if soft_run:
                gsoft = res["soft"][f].cpu().numpy().reshape(c["N"], c["m"])
                bad = soft_mismatch(gsoft, soft)
                assert not bad.any(), (f"{what}: soft: {int(bad.sum())} entries off, worst dln "
                                       f"{np.abs(gsoft - soft)[bad].max(initial=0):.2e}")


def test_invariance_slots_graph_batch(dev):
    name = "C2"
    c = synth.CONFIGS[name]
    _, llr, _ = config_inputs(name, 0, 160)
    code = gpu_code(name)
    x = torch.from_numpy(llr).to(dev)
    base = code.decode(x, c["max_iters"])
    variants = [dict(slots=1), dict(slots=7), dict(slots=160), dict(use_graph=-1, slots=13)]
    for kw in variants:
        o = code.decode(x, c["max_iters"], **kw)
        torch.cuda.synchronize()
        for k in ("hard", "ok", "iters"):
            assert torch.equal(o[k], base[k]), (kw, k)
    sub = torch.arange(17, 160, 9)
    o = code.decode(x[sub].contiguous(), c["max_iters"])
    for k in ("hard", "ok", "iters"):
        assert torch.equal(o[k], base[k][sub.to(dev)]), k
    again = code.decode(x, c["max_iters"])
    for k in ("hard", "ok", "iters"):
        assert torch.equal(again[k], base[k])


def test_workspace_accounting(dev):
    code = gpu_code("C2")
    sb = code.slot_bytes
    c = synth.CONFIGS["C2"]
    assert sb >= 2 * code.E * c["q"] * 4  # the two message sets of a resident frame
    w1, wbig = code.workspace_bytes(1), code.workspace_bytes(1 << 20)
    assert sb <= w1 < 2 * sb and wbig > w1
    S = round((wbig - w1) / sb) + 1  # resident clusters
    assert S >= 100 and S * sb <= wbig <= S * sb + 64 * 1024


def test_caller_workspace_concurrent_streams(dev):
    """nbldpc_decode_opts_t::workspace: decodes with their own workspaces on two streams at once give
    the same results as the handle-workspace decode; a too-small workspace is rejected."""
    import paper_1008_4370_b200 as nb

    name = "C2"
    c = synth.CONFIGS[name]
    _, llr, _ = config_inputs(name, 0, 600)
    x = torch.from_numpy(llr).to(dev)
    code = gpu_code(name)
    base = code.decode(x, c["max_iters"])
    torch.cuda.synchronize()
    halves = (x[:300].contiguous(), x[300:].contiguous())
    nbytes = code.workspace_bytes(300)
    wss = [torch.empty(nbytes + 256, dtype=torch.uint8, device=dev) for _ in range(2)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = []
    for h, ws, s in zip(halves, wss, streams):
        with torch.cuda.stream(s):
            outs.append(code.decode(h, c["max_iters"], workspace=ws, stream=s))
    torch.cuda.synchronize()
    for k in ("hard", "ok", "iters"):
        assert torch.equal(torch.cat([outs[0][k], outs[1][k]]), base[k]), k
    with pytest.raises(nb.NbldpcError):
        code.decode(halves[0], c["max_iters"], workspace=wss[0][: nbytes // 2])
    with pytest.raises(nb.NbldpcError):  # not on the cluster kernel
        code.decode(halves[0], c["max_iters"], workspace=wss[0], vn_algorithm=1)



def test_decode_host_matches_device(dev):
    name = "C5"
    c = synth.CONFIGS[name]
    _, llr, _ = config_inputs(name, 0, 96, point=4)
    code = gpu_code(name)
    d = code.decode(torch.from_numpy(llr).to(dev), c["max_iters"])
    h = code.decode_host(torch.from_numpy(llr).pin_memory(), c["max_iters"])
    for k in ("hard", "ok", "iters"):
        assert torch.equal(d[k].cpu(), h[k])


def test_soft_and_events_outputs(dev):
    name = "C1"
    c = synth.CONFIGS[name]
    _, llr, _ = config_inputs(name, 0, 64)
    code = gpu_code(name)
    out = code.decode(torch.from_numpy(llr).to(dev), 1, early_stop=False, want_soft=True, want_events=True)
    ref = oracle_code(name).lf_decode_batch(llr, 1, early_stop=False, want_soft=True)
    soft = out["soft"].cpu().numpy()
    big = ref["soft"] > -5.0
    assert np.abs(soft[big] - ref["soft"][big]).max() <= 1e-3
    assert int(out["events"].sum()) == 0
    assert (out["iters"].cpu().numpy() == 1).all()


def test_binary_code_and_small_fields(dev):
    import paper_1008_4370_b200 as nb

    for m, poly, N, k in [(1, 0x3, 48, 4), (3, 0xB, 24, 6), (5, 0x25, 40, 4), (7, 0x89, 16, 4)]:
        M, rows, cols, coeffs = synth.make_regular_code(N, k, m, 50 + m)
        code = nb.Code(m, poly, M, N, rows, cols, coeffs)
        ocode = oracle.Code(oracle.Field(m, poly), M, N, rows, cols, coeffs)
        llr = synth.awgn_llr(N * m, 0, 48, synth.sigma2_for(2.0, 1 - 2 / k), 77 + m)
        out = code.decode(torch.from_numpy(llr).to(dev), 20)
        ref = ocode.lf_decode_batch(llr, 20)
        assert_stable_parity(ocode.lf_decode_batch, llr, {k: v.cpu().numpy() for k, v in out.items()}, ref, 20,
                             what=f"m={m}")


def test_edge_cases_and_errors(dev):
    import paper_1008_4370_b200 as nb

    name = "C1"
    c = synth.CONFIGS[name]
    code = gpu_code(name)
    _, llr, _ = config_inputs(name, 0, 1)
    x = torch.from_numpy(llr).to(dev)
    o = code.decode(x, 1)
    ref = oracle_code(name).lf_decode_batch(llr, 1)
    assert o["iters"].item() == 1 and np.array_equal(o["hard"].cpu().numpy(), ref["hard"])
    with pytest.raises(nb.NbldpcError):
        code.decode(x, 0)
    M, rows, cols, coeffs = synth.config_code(name)
    with pytest.raises(nb.NbldpcError) as ei:
        nb.Code(2, 0x5, M, c["N"], rows, cols, coeffs)  # x^2+1 not primitive
    assert ei.value.status == -2
    with pytest.raises(nb.NbldpcError) as ei:
        nb.Code(2, 0x7, M, c["N"] + 1, rows, cols, coeffs)  # a column of weight 0
    assert ei.value.status == -3
    bad = coeffs.copy()
    bad[0] = 4
    with pytest.raises(nb.NbldpcError) as ei:
        nb.Code(2, 0x7, M, c["N"], rows, cols, bad)
    assert ei.value.status == -1


def _irregular_code(N, degs, m, seed):
    """Column weight 2, check degrees `degs` (sum = 2N): socket matching with rejection of repeats."""
    rng = np.random.default_rng(seed)
    M = len(degs)
    for _ in range(1000):
        sockets = np.repeat(np.arange(M), degs)
        var_of = np.repeat(np.arange(N), 2)[rng.permutation(2 * N)]
        pairs = set()
        ok = True
        for c, v in zip(sockets, var_of):
            if (c, v) in pairs:
                ok = False
                break
            pairs.add((c, v))
        if ok:
            coeffs = rng.integers(1, 1 << m, size=2 * N)
            order = np.lexsort((var_of, sockets))
            return M, sockets[order].astype(np.int32), var_of[order].astype(np.int32), coeffs[order].astype(np.int32)
    raise RuntimeError("no simple graph found")


@pytest.mark.parametrize("vn", [0, 1])
def test_irregular_check_degrees_and_cycle_codes(dev, vn):
    """Check degrees that are not a power of two (padding edge slots) and degree-2 checks."""
    import paper_1008_4370_b200 as nb

    cases = [(4, 0x13, 40, [3, 5, 4, 6, 2, 3, 5, 4, 3, 5, 4, 6, 2, 3, 5, 4, 3, 3], 11),
             (6, 0x43, 24, [2] * 24, 12),
             (8, 0x11D, 36, [6, 7, 5, 6, 6, 7, 5, 6, 6, 7, 5, 6][:12], 13)]
    for m, poly, N, degs, seed in cases:
        degs = list(degs)
        if sum(degs) != 2 * N:  # adjust the last degree so that the sockets match
            degs[-1] += 2 * N - sum(degs)
        M, rows, cols, coeffs = _irregular_code(N, degs, m, seed)
        code = nb.Code(m, poly, M, N, rows, cols, coeffs)
        ocode = oracle.Code(oracle.Field(m, poly), M, N, rows, cols, coeffs)
        llr = synth.awgn_llr(N * m, 0, 40, synth.sigma2_for(2.5, 0.5), 90 + m)
        out = code.decode(torch.from_numpy(llr).to(dev), 15, vn_algorithm=vn)
        torch.cuda.synchronize()
        ref = ocode.lf_decode_batch(llr, 15)
        assert_stable_parity(ocode.lf_decode_batch, llr, {k: v.cpu().numpy() for k, v in out.items()}, ref, 15,
                             what=f"m={m} degs {degs[:4]}")


def test_largest_check_team_and_empty_batches(dev):
    """The largest geometry (GF(256), k = 32: 512 threads per check, the 512-thread kernel variant)
    against the oracle, both VN algorithms; an empty batch is rejected as documented (frames >= 1)."""
    import paper_1008_4370_b200 as nb

    m, N, k = 8, 128, 32
    M, rows, cols, coeffs = synth.make_regular_code(N, k, m, 777)
    code = nb.Code(m, 0x11D, M, N, rows, cols, coeffs)
    ocode = oracle.Code(oracle.Field(m, 0x11D), M, N, rows, cols, coeffs)
    llr = synth.awgn_llr(N * m, 0, 6, synth.sigma2_for(4.5, 1 - 2 / k), 778)
    ref = ocode.lf_decode_batch(llr, 15)
    twin = ocode.lf_decode_batch(llr, 15, f32=True)
    stable = (ref["hard"] == twin["hard"]).all(1) & (ref["iters"] == twin["iters"])
    assert stable.sum() >= 4
    for vn in (0, 1):
        out = code.decode(torch.from_numpy(llr).to(dev), 15, vn_algorithm=vn)
        hard, it = out["hard"].cpu().numpy(), out["iters"].cpu().numpy()
        for f in np.where(stable)[0]:
            assert np.array_equal(hard[f], ref["hard"][f]) and it[f] == ref["iters"][f], (vn, f)
    h = torch.zeros((1, N), dtype=torch.uint8, device=dev)
    o = torch.zeros(1, dtype=torch.uint8, device=dev)
    i = torch.zeros(1, dtype=torch.int32, device=dev)
    x = torch.zeros((1, N * m), device=dev)
    L = nb.lib()
    assert L.nbldpc_decode(code._h, x.data_ptr(), 0, 10, h.data_ptr(), o.data_ptr(), i.data_ptr(), None) == -1
    with pytest.raises(ValueError):
        code.decode(torch.zeros((0, N * m), device=dev), 10)


def test_saturated_and_erased_channels(dev):
    """Degenerate channels through the hot path: saturated LLRs (|L| = 1e4, tanh = +-1 exactly) decode
    the sent codeword at the first iteration; all-zero LLRs (an erasure channel, uniform prior) make
    every message neutral, so the decision is the all-zero word, a codeword, at iteration 1 -- the same
    as the oracle in both cases."""
    name = "C3"
    c = synth.CONFIGS[name]
    _, _, xs = config_inputs(name, 0, 8)
    bits = synth.symbols_to_bits(xs, c["m"]).astype(np.float32)
    sat = (1.0 - 2.0 * bits) * 1.0e4
    era = np.zeros_like(sat)
    code = gpu_code(name)
    ocode = oracle_code(name)
    for llr, want in ((sat, xs.astype(np.uint8)), (era, np.zeros_like(xs, dtype=np.uint8))):
        for vn in (0, 1):
            out = code.decode(torch.from_numpy(np.ascontiguousarray(llr)).to(dev), c["max_iters"], vn_algorithm=vn,
                              want_events=True)
            assert (out["iters"] == 1).all() and (out["ok"] == 1).all()
            assert np.array_equal(out["hard"].cpu().numpy(), want)
        ref = ocode.lf_decode_batch(llr, c["max_iters"])
        assert np.array_equal(ref["hard"], want) and (ref["iters"] == 1).all()
