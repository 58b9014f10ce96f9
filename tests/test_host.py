"""Host-side tests that need no GPU: the C-ABI library loads and exports every symbol the
header declares, argument validation (which precedes any CUDA call, include/nbldpc.h), and
the multi-process sharding / counter reduction of the N>1 path over gloo (world size 2)."""
import ctypes
import os
import socket

import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def L():
    import paper_1008_4370_b200 as nb

    return nb.lib()


def test_library_exports_every_header_symbol(L):
    import paper_1008_4370_b200 as nb

    syms = nb.header_symbols()
    for must in ("nbldpc_code_create", "nbldpc_decode", "nbldpc_destroy"):
        assert must in syms
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    # the library's device code is an sm_100a cubin
    import shutil
    import subprocess

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if os.path.exists(tool):
        out = subprocess.run([tool, "--list-elf", nb._build.LIB], capture_output=True, text=True).stdout
        assert "sm_100a" in out, out


def _create(L, m, poly, M, N, rows, cols, coeffs):
    r = np.ascontiguousarray(rows, np.int32)
    c = np.ascontiguousarray(cols, np.int32)
    h = np.ascontiguousarray(coeffs, np.uint16)
    out = ctypes.c_void_p()
    st = L.nbldpc_code_create(m, poly, M, N, r.size, r.ctypes.data, c.ctypes.data, h.ctypes.data, ctypes.byref(out))
    return st, out


def test_status_strings(L):
    for s, txt in [(0, b"ok"), (-1, b"invalid argument"), (-2, b"polynomial"), (-3, b"unsupported"),
                   (-4, b"CUDA"), (-5, b"memory")]:
        assert txt in L.nbldpc_status_string(s)


def test_code_create_validation_without_gpu(L):
    """Every validation error is reported before the library touches the device."""
    M, rows, cols, coeffs = synth.config_code("C1")
    N = 16
    assert _create(L, 2, 0x5, M, N, rows, cols, coeffs)[0] == -2  # x^2+1 not primitive
    assert _create(L, 2, 0x13, M, N, rows, cols, coeffs)[0] == -2  # wrong degree
    assert _create(L, 0, 0x3, M, N, rows, cols, coeffs)[0] == -1  # m out of range
    assert _create(L, 9, 0x211, M, N, rows, cols, coeffs)[0] == -1
    bad = coeffs.copy()
    bad[3] = 4
    assert _create(L, 2, 0x7, M, N, rows, cols, bad)[0] == -1  # coefficient outside GF(4)*
    bad[3] = 0
    assert _create(L, 2, 0x7, M, N, rows, cols, bad)[0] == -1
    badr = rows.copy()
    badr[0] = M
    assert _create(L, 2, 0x7, M, N, badr, cols, coeffs)[0] == -1  # row out of range
    assert _create(L, 2, 0x7, M, N + 1, rows, cols, coeffs)[0] == -3  # a weight-0 column (variable N)
    hv = np.arange(17, dtype=np.int32)  # a weight-17 column: 17 extra rows of degree 2 over variables 0 and 1
    r17 = np.concatenate([rows, M + hv, M + hv])
    c17 = np.concatenate([cols, np.zeros(17, np.int32), np.ones(17, np.int32)])
    h17 = np.concatenate([coeffs, np.ones(34, coeffs.dtype)])
    assert _create(L, 2, 0x7, M + 17, N, r17, c17, h17)[0] == -3
    dup_r = np.concatenate([rows, rows[:1]])
    dup_c = np.concatenate([cols, cols[:1]])
    dup_h = np.concatenate([coeffs, coeffs[:1]])
    assert _create(L, 2, 0x7, M, N, dup_r, dup_c, dup_h)[0] == -3  # duplicate (row, col)
    # a row of degree 1: column 0 moved entirely into its own extra row
    M2, r2, c2, h2 = M + 1, rows.copy(), cols.copy(), coeffs.copy()
    r2[np.where(c2 == 0)[0][0]] = M
    assert _create(L, 2, 0x7, M2, N, r2, c2, h2)[0] == -3
    out = ctypes.c_void_p()
    assert L.nbldpc_code_create(2, 0x7, M, N, len(rows), None, None, None, ctypes.byref(out)) == -1


def test_null_handles_are_rejected(L):
    L.nbldpc_destroy(None)  # no-op
    assert L.nbldpc_decode(None, None, 1, 1, None, None, None, None) == -1
    assert L.nbldpc_code_info(None, None, None, None, None, None) == -1
    assert L.nbldpc_slot_bytes(None) == 0
    assert L.nbldpc_workspace_bytes(None, 10) == 0
    # every decode entry point rejects a NULL handle before touching the device
    assert L.nbldpc_decode_ex(None, None, 1, 1, None, None, None, None, None) == -1
    assert L.nbldpc_decode_pmf(None, None, 1, 1, None, None, None, None, None) == -1
    assert L.nbldpc_decode_host(None, None, 1, 1, None, None, None, None, None) == -1
    assert L.nbldpc_decode_pmf_host(None, None, 1, 1, None, None, None, None, None) == -1
    assert L.nbldpc_step(None, None, 1, 0, None, None, None, None, None, 0, None) == -1
    n = ctypes.c_longlong()
    assert L.nbldpc_last_decode_launches(None, ctypes.byref(n)) == -1


def test_frame_range_partitions_frames():
    from paper_1008_4370_b200 import shard

    # weak: F per rank
    seen = []
    for r in range(8):
        a, b = shard.frame_range(r, 8, 2048, "weak")
        seen.extend(range(a, b))
    assert seen == list(range(8 * 2048))
    # strong: a fixed global batch in contiguous 256-frame-chunk-aligned shards
    for F, G in ((16384, 1), (16384, 2), (16384, 4), (16384, 8), (65536, 8), (1000, 3), (300, 2), (4096, 3)):
        rs = [shard.frame_range(r, G, F, "strong") for r in range(G)]
        assert rs[0][0] == 0 and rs[-1][1] == F
        assert all(rs[i][1] == rs[i + 1][0] for i in range(G - 1))
        assert all(a % 256 == 0 for a, _ in rs)
        if F % (256 * G) == 0:
            assert all(b - a == F // G for a, b in rs)
    with pytest.raises(ValueError):
        shard.frame_range(2, 2, 16)
    with pytest.raises(ValueError):
        shard.frame_range(0, 2, 16, "diagonal")


def test_error_counts_against_sent_codeword():
    from paper_1008_4370_b200 import shard

    hard = torch.zeros((4, 5), dtype=torch.uint8)
    hard[1, 2] = 0b101  # one symbol, two bits wrong, frame flagged converged -> undetected
    hard[2, 0], hard[2, 4] = 1, 0xFF  # two symbols, 9 bits
    ok = torch.tensor([1, 1, 0, 0], dtype=torch.uint8)
    c = shard.error_counts(hard, ok, events=torch.tensor([0, 2, 0, 1], dtype=torch.int32))
    assert c == {"frames": 4, "ok": 2, "frame_err": 2, "sym_err": 3, "bit_err": 11, "undetected": 1, "events": 3}
    sent = hard.clone()
    c = shard.error_counts(hard, ok, sent)
    assert c["frame_err"] == c["sym_err"] == c["bit_err"] == c["undetected"] == 0


def test_llr_shards_do_not_depend_on_sharding():
    """A frame's LLRs depend only on its global index (chunk-keyed Philox), so a rank's shard
    equals the same rows of a single-process batch."""
    whole = synth.config_llr("C5", 0, 600, point=3)
    for world in (2, 3):
        per = 600 // world
        parts = [synth.config_llr("C5", r * per, per, point=3) for r in range(world)]
        assert np.array_equal(np.concatenate(parts), whole[: per * world])
    for world in (2, 3):  # strong-scaling shards (chunk-aligned)
        from paper_1008_4370_b200 import shard

        parts = [synth.config_llr("C5", *(lambda a, b: (a, b - a))(*shard.frame_range(r, world, 600, "strong")),
                                  point=3) for r in range(world)]
        assert np.array_equal(np.concatenate(parts), whole)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


C1_FRAMES, C1_CHUNK = 60, 16


def _c1_sent(f0, f1):
    from parity import config_inputs

    _, llr, xs = config_inputs("C1", f0, f1 - f0)
    return llr, xs


def _gloo_worker(rank, world, port, q):
    """One rank of the N>1 path on CPU: decode ITS strong-scaling shard of C1 (the fp64 oracle
    stands in for the GPU kernel here; the GPU version is tests/test_gpu_shard.py), count errors
    against the sent codewords, reduce the counter vector and the max time, all-gather the outputs."""
    import torch.distributed as dist

    from paper_1008_4370_b200 import shard
    from parity import oracle_code

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, b = shard.frame_range(rank, world, C1_FRAMES, "strong", chunk=C1_CHUNK)
        llr, xs = _c1_sent(a, b)
        r = oracle_code("C1").lf_decode_batch(llr, synth.CONFIGS["C1"]["max_iters"], nthreads=1)
        hard, ok, it = (torch.from_numpy(np.ascontiguousarray(r[k])) for k in ("hard", "ok", "iters"))
        cnt = shard.error_counts(hard.to(torch.uint8), ok, torch.from_numpy(xs))
        cnt["frame_iters"] = int(it.sum())
        c, t = shard.reduce_stats(cnt, {"ms": 10.0 + rank}, dist)
        sizes = [shard.frame_range(g, world, C1_FRAMES, "strong", chunk=C1_CHUNK) for g in range(world)]
        sizes = [y - x for x, y in sizes]
        g_hard = shard.gather_rows(hard.to(torch.int32), dist, sizes)
        g_ok = shard.gather_rows(ok.to(torch.int32), dist, sizes)
        g_it = shard.gather_rows(it.to(torch.int32), dist, sizes)
        q.put((rank, c, t, g_hard.numpy(), g_ok.numpy(), g_it.numpy()))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_sharded_decode_and_reduction():
    """Two gloo ranks decode their shards; the all-gathered outputs and the reduced counters are
    identical to a single-process decode of the whole batch."""
    import torch.multiprocessing as mp

    from paper_1008_4370_b200 import shard
    from parity import oracle_code

    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda x: x[0])
    llr, xs = _c1_sent(0, C1_FRAMES)
    r = oracle_code("C1").lf_decode_batch(llr, synth.CONFIGS["C1"]["max_iters"], nthreads=1)
    want = shard.error_counts(torch.from_numpy(r["hard"].astype(np.uint8)), torch.from_numpy(r["ok"]),
                              torch.from_numpy(xs))
    want["frame_iters"] = int(r["iters"].sum())
    for _, c, t, gh, gok, git in res:
        assert c == want
        assert t == {"ms": 11.0}
        assert np.array_equal(gh, r["hard"]) and np.array_equal(gok, r["ok"]) and np.array_equal(git, r["iters"])
    assert want["frame_err"] > 0  # the sample exercises the error counters (C1 at 2 dB has failures)
