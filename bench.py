#!/usr/bin/env python
"""Benchmark of the B200 Log-Fourier SP decoder (arXiv:1008.4370) -- one JSON line on rank 0.

A "step" is one nbldpc_decode of the whole batch: every frame of the workload runs
the full hot path (channel spectrum, variable node, tentative decision, check node,
syndrome, early termination) until it stops.  Workload at N=1: BASELINE.json
configs[1] (C2: GF(64), (2,4)-regular, N=1024, 4096 all-zero-codeword frames,
BPSK/AWGN Eb/N0 = 1.0 dB, 50 iterations with early stop), synthetic seeded inputs.

metric = sum_f K_bits * iters_used_f / T  (decoded info bits per second per iteration),
K_bits = N m (1 - 2/k).  Multi-GPU (torchrun): weak scaling, each rank decodes its own
4096-frame shard (global frame indices rank*F ..), NCCL only for the final counter /
timing reductions.  L2 is flushed (256 MiB write) before every timed step.

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
    mufu = 2 * E * q + N * q                        # ex2 of every VN input entry, lg2 of every output, ex2 of W_a
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


def cpu_oracle_run(cfg, point, frame0, nframes, threads=None, inp="llr", ebn0=None, symbol_out=False, algorithm="lf"):
    """Times the oracle (as it stands) on frames frame0.. of the workload; returns (value, seconds, iters)."""
    import oracle

    M, rows, cols, coeffs = synth.config_code(cfg["name"])
    code = oracle.Code(oracle.Field(cfg["m"], cfg["poly"]), M, cfg["N"], rows, cols, coeffs)
    x = channel_input(cfg, inp, point, ebn0, frame0, nframes)
    nt = threads or os.cpu_count() or 1
    t0 = time.perf_counter()
    if algorithm == "logsp":
        r = code.ls_decode_batch(x, cfg["max_iters"], pmf=inp == "pmf", nthreads=nt)
    else:
        dec = code.lf_decode_batch_pmf if inp == "pmf" else code.lf_decode_batch
        r = dec(x, cfg["max_iters"], nthreads=nt, want_post=symbol_out)
    dt = time.perf_counter() - t0
    it = int(r["iters"].sum())
    return info_bits(cfg) * it / dt, dt, it, nt


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    vals, dts = [], []
    nframes = args.ref_frames
    for i in range(args.warmup + args.steps):
        v, dt, it, nt = cpu_oracle_run(cfg, args.point, i * nframes, nframes, inp=args.input, ebn0=args.ebn0,
                                       symbol_out=args.symbol_out, algorithm=args.algorithm)
        if i >= args.warmup:
            vals.append(v)
            dts.append(dt)
    total_bits = sum(v * d for v, d in zip(vals, dts))
    value = total_bits / sum(dts)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(dts) / len(dts),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(cfg, args.point, args.input, args.ebn0), "frames_per_step": nframes,
                   "sample": f"{nframes} frames per step (frames i*{nframes}.. of the seeded stream)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nt, "kind": "oracle",
                         "sample": f"{nframes} frames per step x {args.steps} steps, fp64 C oracle, OpenMP"},
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
    ap.add_argument("--config", default="C2")
    ap.add_argument("--point", type=int, default=0)
    ap.add_argument("--frames", type=int, default=0, help="frames per rank (default: the config's)")
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
    ap.add_argument("--ref-frames", type=int, default=32)
    ap.add_argument("--cpu-frames", type=int, default=64)
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

    F = args.frames or cfg["frames"]
    f0, f1 = shard.frame_range(rank, world, F)
    M, rows, cols, coeffs = synth.config_code(cfg["name"])
    code = nb.Code(cfg["m"], cfg["poly"], M, cfg["N"], rows, cols, coeffs)
    pmf_in = args.input == "pmf"
    vn = 1 if (args.symbol_out and pmf_in) else args.vn  # pmf + symbol outputs run the slot-pass kernel
    llr_np = channel_input(cfg, args.input, args.point, args.ebn0, f0, f1 - f0)
    llr_host = torch.from_numpy(llr_np).pin_memory()
    llr = llr_host.to(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    kw = dict(slots=args.slots, use_graph=args.graph, want_post=args.symbol_out, vn_algorithm=vn,
              algorithm=1 if args.algorithm == "logsp" else 0, message_format=1 if args.msg == "f16" else 0)
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
    step_ms, iters_sum, launches, ok_sum = [], 0, 0, 0
    for _ in range(args.steps):
        flush.fill_(1)  # L2 flush (untimed)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        out = decode(llr, cfg["max_iters"], **kw)
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        iters_sum += int(out["iters"].sum().item())
        ok_sum += int(out["ok"].sum().item())
        launches += code.last_decode_launches()
    barrier()
    clk = clocks.stop()

    # end to end through the host-buffer C-ABI entry (H2D + decode + D2H inside the timed region)
    e2e_ms, e2e_iters, d2h = 0.0, 0, F * cfg["N"] + F + 4 * F
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
        kw.pop("want_post")
        code.decode_host(llr_host, cfg["max_iters"], **kw)
        barrier()
        for _ in range(args.steps):
            flush.fill_(1)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            hout = code.decode_host(llr_host, cfg["max_iters"], **kw)
            e2e_ms += 1e3 * (time.perf_counter() - t0)
            e2e_iters += int(hout["iters"].sum())
        barrier()

    cnt, tim = shard.reduce_stats(
        {"frame_iters": iters_sum, "ok": ok_sum, "frames": F * args.steps, "launches": launches,
         "e2e_frame_iters": e2e_iters},
        {"ms": sum(step_ms), "e2e_ms": e2e_ms}, dist, device=dev)
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return 0

    value = info_bits(cfg) * cnt["frame_iters"] / (tim["ms"] * 1e-3)
    traffic = None
    if os.path.exists(args.traffic):
        try:
            key = (f"{cfg['name']}:vn{vn}" + (":pmf" if pmf_in else "") + (":sym" if args.symbol_out else "")
                   + (":f16" if args.msg == "f16" else "") + (":logsp" if args.algorithm == "logsp" else ""))
            traffic = json.load(open(args.traffic)).get(key)
        except (OSError, ValueError):
            traffic = None
    # this rank's kernel: its frame-iterations over its own device time
    roof = roofline(cfg, vn, iters_sum, sum(step_ms) * 1e-3, traffic, args.input, args.symbol_out, args.algorithm,
                    args.msg)
    roof["kernel"] = ("lf_cluster_kernel (one launch per step + a 1-block setup kernel; "
                      "CUDA events around the step)") if vn == 0 else "nb_pass_kernel (slot passes)"
    if args.algorithm == "logsp":
        roof["kernel"] = "ls_frame_kernel (conventional Log-SP, one CTA per frame; one launch per step)"
    elif vn == 2 or cfg["j"] != 2:
        roof["kernel"] = "lfg_frame_kernel (general column weight, one CTA per frame; one launch per step)"
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": warm, "ms_per_step": tim["ms"] / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_name(cfg, args.point, args.input, args.ebn0), "frames_per_gpu": F,
                   "global_frames": F * world, "N": cfg["N"], "q": cfg["q"], "k": cfg["k"],
                   "max_iters": cfg["max_iters"], "vn_algorithm": ["separable", "direct", "general"][vn],
                   "column_weight": cfg["j"],
                   "input": args.input, "symbol_outputs": bool(args.symbol_out), "algorithm": args.algorithm,
                   "messages": args.msg,
                   "parallelism": f"frames sharded over {world} GPU(s), no collective in the loop",
                   "l2": "flushed (256 MiB write) before every timed step",
                   "slots": args.slots or "default", "mean_iters": cnt["frame_iters"] / cnt["frames"],
                   "frame_error_rate": 1.0 - cnt["ok"] / cnt["frames"]},
        "roofline": roof,
        "gpu_launches": int(cnt["launches"]),
        "clocks": clk,
    }
    if not args.no_e2e:
        line["e2e"] = {"value": info_bits(cfg) * cnt["e2e_frame_iters"] / (tim["e2e_ms"] * 1e-3), "unit": UNIT,
                       "h2d_bytes_per_step": int(llr_np.nbytes), "d2h_bytes_per_step": int(d2h)}
    if not args.no_cpu_baseline and world == 1:
        v, dt, it, nt = cpu_oracle_run(cfg, args.point, 0, args.cpu_frames, inp=args.input, ebn0=args.ebn0,
                                       symbol_out=args.symbol_out, algorithm=args.algorithm)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": nt, "kind": "oracle",
                                "sample": f"first {args.cpu_frames} frames of the workload, {it} frame-iterations, "
                                          f"{dt:.1f} s, fp64 C oracle with OpenMP over frames"}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
