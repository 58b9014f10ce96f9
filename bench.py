#!/usr/bin/env python
"""Benchmark of the B200 Log-Fourier SP decoder (arXiv:1008.4370) -- one JSON line on rank 0.

A "step" is one nbldpc_decode of the whole batch: every frame of the workload runs
the full hot path (channel spectrum, variable node, tentative decision, check node,
syndrome, early termination) until it stops.  Workload (default): BASELINE.json
configs[3], the configuration the metric "(1/2/4/8 B200)" is quoted on -- C4: GF(256),
(2,16)-regular, N=2048, a global batch of 16,384 all-zero-codeword frames, BPSK/AWGN
Eb/N0 = 3.5 dB, 30 iterations with early stop; synthetic seeded inputs.  --config picks
another BASELINE config (C1..C5), --point a C5 Eb/N0 point.

metric = sum_f K_bits * iters_used_f / T  (decoded info bits per second per iteration),
K_bits = N m (1 - 2/k).  Multi-GPU (torchrun): strong scaling by default -- the config's
fixed global batch in chunk-aligned contiguous shards (shard.frame_range); --scaling weak
gives every rank F frames.  No collective in the loop; one NCCL all-reduce of the counter
vector (frames, converged, frame / symbol / bit errors against the sent codeword,
undetected errors, iterations, numerical events) and one MAX of the device times after
it.  L2 is flushed (256 MiB write) before every timed step.

--impl reference times the CPU oracle (oracle/, fp64, OpenMP over frames) on a bounded
sample of the same workload; it is the base contract's reference arm for this tier.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "decoded info bits/s per iteration (1/2/4/8 B200) and % of roofline"
UNIT = "info-bit-iterations/s"
# Peaks.  HBM: MEASURED_PEAKS.json (driver-measured copy bandwidth).  SFU (MUFU ex2/lg2)
# and FP32 FMA: 148 SMs x 16 (MUFU) / 128 (FMA) lanes per clock x 1.965 GHz, the guide's unit counts at
# clocks.max.sm; profiles/r01_microbench.log measured 15.85 MUFU and 127.6 FMA per SM-clock.
SMS, CLK = 148, 1.965e9
MUFU_PEAK = SMS * 16 * CLK          # ops/s
FMA_PEAK = SMS * 128 * CLK          # FMA/s
HBM_PEAK_FALLBACK = 6.65e12         # B200_PROFILING.md fallback, used only if MEASURED_PEAKS.json is absent


def hbm_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]) * 1e9, "measured"
    except (OSError, ValueError, KeyError):
        return HBM_PEAK_FALLBACK, "fallback"


def per_frame_iter(cfg, vn, inp="llr", symbol_out=False, algorithm="lf", msg="f32"):
    """Algorithmic work of one frame-iteration: SFU ops, FP32 FMAs, message bytes.
    inp = "pmf": the channel spectrum is a q-vector per variable (read per iteration from the slot
    buffer) instead of m channel terms; symbol_out: + the symbol posterior written per iteration
    and its two WHTs (counted as FMA-pipe ops)."""
    N, q, m = cfg["N"], cfg["q"], cfg["m"]
    E = cfg["j"] * N
    if vn == 2 or cfg["j"] != 2:
        # general kernel: per edge 2 WHTs (W -> w, product -> U) of m q butterflies, the leave-one-out
        # products; per variable the decision sums; messages U and W each written once and read once
        return 2 * E * q, 2 * E * m * q + E * q * cfg["j"] + N * (m + 1) * q, 4 * E * q * 4 + 4 * N * m + N
    if algorithm == "logsp":
        # conventional Log-SP: 3(k-2) q^2-term log-convolutions per check (forward-
        # backward), each input exponentiated twice and each output's log once; messages + lambda^0
        Mc = E // cfg["k"]
        return 3 * E * q, Mc * 3 * (cfg["k"] - 2) * q * q, 2 * E * q * 4 + 4 * N * q + N
    # SFU ops: the packed-log format (f16 messages) takes an ex2 of every VN input entry, an lg2 of every
    # output and an ex2 of every W_a entry of the decision; the f32 hot path stores linear messages
    # at q >= 128 and needs one reciprocal per edge (the normalisation) only
    mufu = (2 * E * q + N * q) if (msg == "f16" or cfg["m"] < 7) else E
    if inp == "pmf":  # probability-domain VN: 2 WHTs (m q add/sub each) and a product per entry
        fma = E * q * (2 * m + 1) + N * (m + 1) * q
    else:             # VN (separable / direct) + decision points
        fma = (E * m * q if vn == 0 else E * q * q) + N * (m + 1) * q
    bytes_ = 2 * E * q * (2 if msg == "f16" else 4) + N  # one message set read + written, symbols
    bytes_ += 4 * N * q if inp == "pmf" else 4 * N * m  # channel spectrum / channel terms
    if symbol_out:
        fma += N * q * (2 * m + 1)
        bytes_ += 4 * N * q + N
    return mufu, fma, bytes_


def roofline(cfg, vn, frame_iters, seconds, traffic, inp="llr", symbol_out=False, algorithm="lf", msg="f32"):
    """The slower of the SFU, FP32 and HBM-message-byte bounds (BASELINE.json north_star) for the
    work done; achieved / peak of that resource over the measured kernel time."""
    mufu, fma, byts = per_frame_iter(cfg, vn, inp, symbol_out, algorithm, msg)
    hbm, hbm_src = hbm_peak()
    t = {"alu": max(mufu / MUFU_PEAK, fma / FMA_PEAK), "hbm": byts / hbm}
    bound = max(t, key=t.get)
    n = frame_iters
    comps = {
        "sfu": {"achieved_Tops": mufu * n / seconds / 1e12, "peak_Tops": MUFU_PEAK / 1e12,
                "frac": mufu * n / seconds / MUFU_PEAK},
        "fp32_fma": {"achieved_TFLOPs": 2 * fma * n / seconds / 1e12, "peak_TFLOPs": 2 * FMA_PEAK / 1e12,
                     "frac": fma * n / seconds / FMA_PEAK},
        "hbm_message_bytes": {"achieved_GBs": byts * n / seconds / 1e9, "peak_GBs": hbm / 1e9, "peak_source": hbm_src,
                              "frac": byts * n / seconds / hbm},
    }
    if bound == "hbm":
        r = {"bound": "hbm", "achieved": byts * n / seconds / 1e9, "peak": hbm / 1e9, "unit": "GB/s"}
    elif mufu / MUFU_PEAK >= fma / FMA_PEAK:
        r = {"bound": "alu", "achieved": mufu * n / seconds / 1e12, "peak": MUFU_PEAK / 1e12,
             "unit": "TFLOP/s", "pipe": "SFU (MUFU ex2/lg2 ops, not FLOPs)"}
    else:
        r = {"bound": "alu", "achieved": 2 * fma * n / seconds / 1e12, "peak": 2 * FMA_PEAK / 1e12,
             "unit": "TFLOP/s", "pipe": "FP32 FMA"}
    r["frac"] = r["achieved"] / r["peak"]
    r["traffic"] = traffic
    r["components"] = comps
    r["roofline_info_bits_iter_per_s"] = info_bits(cfg) / max(t.values())
    return r


def channel_input(cfg, inp, point, ebn0, frame0, nframes):
    """LLRs [F][N*m] (BPSK/AWGN) or symbol pmfs [F][N][q] (q-ary orthogonal signalling over AWGN)."""
    if inp == "pmf":
        return synth.config_pmf(cfg["name"], frame0, nframes, ebn0_db=ebn0, point=point)
    return synth.config_llr(cfg["name"], frame0, nframes, ebn0_db=ebn0, point=point)


def info_bits(cfg) -> float:
    return cfg["N"] * cfg["m"] * cfg["rate"]


def workload_name(cfg, point, inp="llr", ebn0=None):
    eb = cfg["ebn0"][point] if ebn0 is None else ebn0
    ch = "BPSK/AWGN bit LLRs" if inp == "llr" else f"{cfg['q']}-ary orthogonal signalling/AWGN symbol pmfs"
    return (f"{cfg['name']}: GF({cfg['q']}) ({cfg['j']},{cfg['k']})-regular N={cfg['N']} rate {cfg['rate']:.4g}, "
            f"{ch}, Eb/N0={eb} dB, max {cfg['max_iters']} iters, early stop, "
            f"{'random' if cfg['codeword'] == 'random' else 'all-zero'} codewords")


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=5)
        sm, smax, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            p = [x.strip() for x in line.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                smax = max(smax, float(p[1]))
            except ValueError:
                continue
            for n, v in zip(names, p[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return None
        loaded = [x for x in sm if x > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# oracle cost is ~E q^2 exponentials per frame-iteration: cap the iterations of the CPU samples of the
# GF(256) configs so that a sample stays within seconds (measured: C4 4.9 s, C3 1.4 s, C2 0.2 s, C5 0.08 s
# per frame-iteration per core); the metric counts the iterations actually run
ORACLE_ITER_CAP = {"C3": 2, "C4": 1}


def cpu_oracle_run(cfg, point, frame0, nframes, threads=None, inp="llr", ebn0=None, symbol_out=False, algorithm="lf",
                   max_iters=None):
    """Times the oracle (as it stands) on frames frame0.. of the workload; returns (value, seconds, iters, threads)."""
    import oracle

    M, rows, cols, coeffs = synth.config_code(cfg["name"])
    code = oracle.Code(oracle.Field(cfg["m"], cfg["poly"]), M, cfg["N"], rows, cols, coeffs)
    x = channel_input(cfg, inp, point, ebn0, frame0, nframes)
    nt = threads or os.cpu_count() or 1
    iters = max_iters or cfg["max_iters"]
    t0 = time.perf_counter()
    if algorithm == "logsp":
        r = code.ls_decode_batch(x, iters, pmf=inp == "pmf", nthreads=nt)
    else:
        dec = code.lf_decode_batch_pmf if inp == "pmf" else code.lf_decode_batch
        r = dec(x, iters, nthreads=nt, want_post=symbol_out)
    dt = time.perf_counter() - t0
    it = int(r["iters"].sum())
    return info_bits(cfg) * it / dt, dt, it, nt


def oracle_sample(cfg, nframes, iters_cap):
    cap = min(cfg["max_iters"], iters_cap or ORACLE_ITER_CAP.get(cfg["name"], cfg["max_iters"]))
    return cap, (f"{nframes} frames of the workload, at most {cap} of its {cfg['max_iters']} iterations each"
                 + (" (the fp64 oracle costs seconds per frame-iteration here)" if cap < cfg["max_iters"] else ""))


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    vals, dts = [], []
    cores = os.cpu_count() or 1
    nframes = args.ref_frames or min(32, max(8, cores))
    cap, sample = oracle_sample(cfg, nframes, args.ref_iters)
    nt = cores
    for i in range(args.warmup + args.steps):
        v, dt, it, nt = cpu_oracle_run(cfg, args.point, i * nframes, nframes, inp=args.input, ebn0=args.ebn0,
                                       symbol_out=args.symbol_out, algorithm=args.algorithm, max_iters=cap)
        if i >= args.warmup:
            vals.append(v)
            dts.append(dt)
    total_bits = sum(v * d for v, d in zip(vals, dts))
    value = total_bits / sum(dts)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(dts) / len(dts),
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(cfg, args.point, args.input, args.ebn0), "frames_per_step": nframes,
                   "sample": f"each step: {sample} (frames i*{nframes}.. of the seeded stream)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nt, "kind": "oracle",
                         "sample": f"{sample}, x {args.steps} steps, fp64 C oracle, OpenMP over frames"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4",
                    help="BASELINE.json config (default C4, the 1/2/4/8-GPU configuration the metric is quoted on)")
    ap.add_argument("--point", type=int, default=0)
    ap.add_argument("--frames", type=int, default=0,
                    help="strong scaling: the global batch (default: the config's); weak: frames per rank")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the config's fixed global batch split over the ranks (default); weak: F per rank")
    ap.add_argument("--slots", type=int, default=0)
    ap.add_argument("--graph", type=int, default=0, help="direct path only: 0 graph, -1 host loop")
    ap.add_argument("--vn", type=int, default=0,
                    help="0 separable (default), 1 direct q^2 convolution, 2 general column weight kernel")
    ap.add_argument("--input", default="llr", choices=["llr", "pmf"],
                    help="llr: BPSK bit LLRs (nbldpc_decode); pmf: symbol pmfs (nbldpc_decode_pmf)")
    ap.add_argument("--ebn0", type=float, default=None, help="override the config's Eb/N0 (dB)")
    ap.add_argument("--symbol-out", action="store_true", help="also output the symbol posterior and MAP decision")
    ap.add_argument("--algorithm", default="lf", choices=["lf", "logsp"],
                    help="lf: Log-Fourier SP (the hot path); logsp: the conventional Log-SP it is compared with")
    ap.add_argument("--msg", default="f32", choices=["f32", "f16"],
                    help="message storage: f32 (default) or f16 (half the message bytes; evaluated by FER)")
    ap.add_argument("--ref-frames", type=int, default=0, help="reference arm: frames per step (default: cores)")
    ap.add_argument("--ref-iters", type=int, default=0, help="reference arm: iteration cap (default per config)")
    ap.add_argument("--cpu-frames", type=int, default=0, help="cpu_baseline sample frames (default: cores)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--traffic", default=os.path.join(ROOT, "profiles", "traffic.json"))
    args = ap.parse_args()
    cfg = synth.CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch

    from paper_1008_4370_b200 import shard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)

    import paper_1008_4370_b200 as nb

    Fcfg = args.frames or cfg["frames"]
    f0, f1 = shard.frame_range(rank, world, Fcfg, args.scaling)
    F = f1 - f0
    if F < 1:
        raise SystemExit(f"rank {rank}: empty shard of {Fcfg} frames over {world} ranks")
    global_frames = Fcfg if args.scaling == "strong" else Fcfg * world
    M, rows, cols, coeffs = synth.config_code(cfg["name"])
    code = nb.Code(cfg["m"], cfg["poly"], M, cfg["N"], rows, cols, coeffs)
    pmf_in = args.input == "pmf"
    vn = 1 if (args.symbol_out and pmf_in) else args.vn  # pmf + symbol outputs run the slot-pass kernel
    llr_np = channel_input(cfg, args.input, args.point, args.ebn0, f0, F)
    llr_host = torch.from_numpy(llr_np).pin_memory()
    llr = llr_host.to(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    logsp = args.algorithm == "logsp"
    kw = dict(slots=args.slots, use_graph=args.graph, want_post=args.symbol_out, vn_algorithm=vn,
              algorithm=1 if logsp else 0, message_format=1 if args.msg == "f16" else 0,
              want_events=not logsp)
    decode = code.decode_pmf if pmf_in else code.decode

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    warm = max(3, args.warmup)
    for _ in range(warm):
        out = decode(llr, cfg["max_iters"], **kw)
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    step_ms, launches = [], 0
    cnt = {k: 0 for k in shard.COUNTERS}
    for _ in range(args.steps):
        flush.fill_(1)  # L2 flush (untimed)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        out = decode(llr, cfg["max_iters"], **kw)
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        # outside the timed region: counters against the sent (all-zero) codeword
        for k, v in shard.error_counts(out["hard"], out["ok"], None, out.get("events")).items():
            cnt[k] += v
        cnt["frame_iters"] += int(out["iters"].to(torch.int64).sum().item())
        launches += code.last_decode_launches()
    barrier()
    clk = clocks.stop()
    cnt["launches"] = launches
    my_iters = cnt["frame_iters"]

    # end to end through the host-buffer C-ABI entry (H2D + decode + D2H inside the timed region)
    e2e_ms, e2e_iters, d2h = 0.0, 0, F * cfg["N"] + F + 4 * F
    hkw = {k: v for k, v in kw.items() if k not in ("want_post", "want_events")}
    if not args.no_e2e and pmf_in and not args.symbol_out:
        # through the host-buffer C-ABI entry (pinned pmfs -> device -> decode -> host outputs, all timed)
        hkw = dict(slots=args.slots, vn_algorithm=vn, algorithm=kw["algorithm"])
        code.decode_pmf_host(llr_host, cfg["max_iters"], **hkw)
        barrier()
        for _ in range(args.steps):
            flush.fill_(1)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            hout = code.decode_pmf_host(llr_host, cfg["max_iters"], **hkw)
            e2e_ms += 1e3 * (time.perf_counter() - t0)
            e2e_iters += int(hout["iters"].sum())
        barrier()
    elif not args.no_e2e and (pmf_in or args.symbol_out):
        # through the Python binding: pinned H2D copy of the inputs, decode, D2H of every output
        if args.symbol_out:
            d2h += F * cfg["N"] * (4 * cfg["q"] + 1)
        host_out = {k: torch.empty(v.shape, dtype=v.dtype).pin_memory() for k, v in out.items()}
        dev_in = torch.empty_like(llr)
        barrier()
        for i in range(args.steps + 1):
            flush.fill_(1)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dev_in.copy_(llr_host, non_blocking=True)
            o = decode(dev_in, cfg["max_iters"], **kw)
            for k in o:
                host_out[k].copy_(o[k], non_blocking=True)
            torch.cuda.synchronize()
            if i > 0:  # the first call is an untimed warm-up of the staging path
                e2e_ms += 1e3 * (time.perf_counter() - t0)
                e2e_iters += int(host_out["iters"].sum())
        barrier()
    elif not args.no_e2e:
        code.decode_host(llr_host, cfg["max_iters"], **hkw)
        barrier()
        for _ in range(args.steps):
            flush.fill_(1)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            hout = code.decode_host(llr_host, cfg["max_iters"], **hkw)
            e2e_ms += 1e3 * (time.perf_counter() - t0)
            e2e_iters += int(hout["iters"].sum())
        barrier()
    cnt["e2e_frame_iters"] = e2e_iters

    # ONE all-reduce of the counter vector (SUM) and one of the device times (MAX) -- SURVEY.md 8(e)
    cnt, tim = shard.reduce_stats(cnt, {"ms": sum(step_ms), "e2e_ms": e2e_ms}, dist, device=dev)
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return 0

    value = info_bits(cfg) * cnt["frame_iters"] / (tim["ms"] * 1e-3)
    traffic = None
    if os.path.exists(args.traffic):
        try:
            key = (f"{cfg['name']}:vn{vn}" + (":pmf" if pmf_in else "") + (":sym" if args.symbol_out else "")
                   + (":f16" if args.msg == "f16" else "") + (":logsp" if logsp else ""))
            traffic = json.load(open(args.traffic)).get(key)
        except (OSError, ValueError):
            traffic = None
    # this rank's kernel: its frame-iterations over its own device time
    roof = roofline(cfg, vn, my_iters, sum(step_ms) * 1e-3, traffic, args.input, args.symbol_out, args.algorithm,
                    args.msg)
    roof["kernel"] = ("lf_cluster_kernel (one launch per step + a 1-block setup kernel; "
                      "CUDA events around the step)") if vn == 0 else "nb_pass_kernel (slot passes)"
    if logsp:
        roof["kernel"] = "ls_frame_kernel (conventional Log-SP, one CTA per frame; one launch per step)"
    elif vn == 2 or cfg["j"] != 2:
        roof["kernel"] = "lfg_frame_kernel (general column weight, one CTA per frame; one launch per step)"
    nfr = cnt["frames"]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": warm, "ms_per_step": tim["ms"] / args.steps, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_name(cfg, args.point, args.input, args.ebn0), "frames_per_gpu": F,
                   "global_frames": global_frames, "N": cfg["N"], "q": cfg["q"], "k": cfg["k"],
                   "max_iters": cfg["max_iters"], "vn_algorithm": ["separable", "direct", "general"][vn],
                   "column_weight": cfg["j"],
                   "input": args.input, "symbol_outputs": bool(args.symbol_out), "algorithm": args.algorithm,
                   "messages": args.msg,
                   "parallelism": (f"{args.scaling} scaling: {global_frames} frames in chunk-aligned contiguous "
                                   f"shards over {world} GPU(s), no collective in the loop, one NCCL all-reduce "
                                   f"of the counter vector after it"),
                   "l2": "flushed (256 MiB write) before every timed step",
                   "slots": args.slots or "default", "mean_iters": cnt["frame_iters"] / nfr,
                   "codeword": "all-zero (sent codeword for the error counts)",
                   "frame_error_rate": cnt["frame_err"] / nfr,
                   "symbol_error_rate": cnt["sym_err"] / (nfr * cfg["N"]),
                   "bit_error_rate": cnt["bit_err"] / (nfr * cfg["N"] * cfg["m"]),
                   "undetected_frames": cnt["undetected"], "syndrome_fail_rate": 1.0 - cnt["ok"] / nfr,
                   "numeric_events": cnt["events"], "frames_decoded": nfr},
        "roofline": roof,
        "gpu_launches": int(cnt["launches"]),
        "clocks": clk,
    }
    if not args.no_e2e:
        line["e2e"] = {"value": info_bits(cfg) * cnt["e2e_frame_iters"] / (tim["e2e_ms"] * 1e-3), "unit": UNIT,
                       "h2d_bytes_per_step": int(llr_np.nbytes) * world, "d2h_bytes_per_step": int(d2h) * world}
    if not args.no_cpu_baseline and world == 1:
        n = args.cpu_frames or (os.cpu_count() or 1)
        cap, sample = oracle_sample(cfg, n, 0 if cfg["name"] != "C4" else 2)
        v, dt, it, nt = cpu_oracle_run(cfg, args.point, 0, n, inp=args.input, ebn0=args.ebn0,
                                       symbol_out=args.symbol_out, algorithm=args.algorithm, max_iters=cap)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": nt, "kind": "oracle",
                                "sample": f"first {sample}: {it} frame-iterations, {dt:.1f} s, fp64 C oracle with "
                                          f"OpenMP over frames"}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
