#!/usr/bin/env python
"""bench.py — PPD serving data path on B200 (see DESIGN.md §6 for definitions).

Headline (N=1, BASELINE.json configs[1]): Llama-3-8B-shape random-init bf16 on
one colocated B200; a "step" is one fused decode iteration of B=200 requests at
context ~1024 through ppd_step (the C-ABI seam that replaces
decode_step_time, reference costmodel.cpp:372-379). value = decode tokens/s
(device time, CUDA events on the library's compute stream); e2e = the same
through the C-ABI with host arrays and the H2D/D2H copies inside the timed
region. The interference sweep of configs[1] (colocated full vs append
prefill riding in the decode step) is reported beside it.

--impl reference: the reference has no model (it prices this step with an
analytic formula); its CPU arm here is the CPU port of the same decode step
(oracle/model_oracle.c, kind "port") on all host cores, bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = json.load(open(os.path.join(REPO, "BASELINE.json")))["metric"]
SEED = 20260313
# Dry run of the N > 1 path on a one-GPU box (tests only): every rank and every
# engine node maps to GPU 0 and torch.distributed uses gloo. Never set for a
# measurement: the numbers it prints are not multi-GPU numbers.
SAME_GPU = os.environ.get("PPD_BENCH_SAME_GPU") == "1"


def gpu_of(i: int) -> int:
    return 0 if SAME_GPU else i


def peaks():
    try:
        return json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled (NVML, every 50 ms) during the timed region."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples = []
        self.stop = threading.Event()
        self.err = None

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception as e:  # noqa: BLE001
            self.err = repr(e)
        return self

    def _run(self):
        N = self.N
        while not self.stop.is_set():
            try:
                self.samples.append((N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM),
                                     N.nvmlDeviceGetCurrentClocksEventReasons(self.h)))
            except Exception as e:  # noqa: BLE001
                self.err = repr(e)
            self.stop.wait(0.05)

    def __exit__(self, *a):
        self.stop.set()
        if hasattr(self, "t"):
            self.t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "error": self.err}
        N = self.N
        names = {"hw_slowdown": N.nvmlClocksEventReasonHwSlowdown,
                 "hw_thermal_slowdown": N.nvmlClocksEventReasonHwThermalSlowdown,
                 "sw_thermal_slowdown": N.nvmlClocksEventReasonSwThermalSlowdown,
                 "sw_power_cap": N.nvmlClocksEventReasonSwPowerCap,
                 "hw_power_brake": N.nvmlClocksEventReasonHwPowerBrakeSlowdown}
        reasons = sorted({n for _, r in self.samples for n, bit in names.items() if r & bit})
        sm = [c for c, _ in self.samples]
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(sm)}


# ----------------------------------------------------------------- CPU port
class CpuPortStep:
    """The CPU port (oracle/model_oracle.c, all host threads) of one
    Llama-3-8B-shape decode step of `batch` rows at context `ctx`. One sample
    times a 1-layer and a 2-layer step (bounded: ~1-2 s) and extrapolates
    t = t_head + layers_full * t_layer (t_layer = t2 - t1)."""

    def __init__(self, batch: int, ctx: int, layers_full: int = 32):
        from oracle import oracle as O
        self.O, self.batch, self.ctx, self.layers_full = O, batch, ctx, layers_full
        cfg = O.MoCfg(2, 4096, 32, 8, 128, 14336, 128256, 1e-5, 5e5, 0)
        self.cfg = cfg
        self.m = O.Model(cfg, SEED)
        nbps = (ctx + 1 + 15) // 16
        self.pool = O.KvPool(cfg, batch * nbps)
        rng = np.random.default_rng(1)
        self.pool.data[...] = O.f32_to_bf16((rng.standard_normal(self.pool.data.shape, dtype=np.float32) * 0.5))
        self.bts = np.arange(batch * nbps, dtype=np.int32).reshape(batch, nbps)
        self.toks = rng.integers(0, cfg.vocab, batch).astype(np.int32)

    def sample(self):
        times = {}
        for nl in (1, 2):
            self.m.set_active_layers(nl)
            t0 = time.perf_counter()
            self.m.step(self.pool, [1] * self.batch, [self.ctx] * self.batch, self.toks, self.bts, want_logits=False)
            times[nl] = time.perf_counter() - t0
        t_layer = max(times[2] - times[1], 1e-9)
        t_head = max(times[1] - t_layer, 0.0)
        t_full = t_head + self.layers_full * t_layer
        desc = (f"{self.batch} decode rows at ctx {self.ctx}: a 1- and a 2-layer Llama-3-8B-shape step timed, "
                f"extrapolated to {self.layers_full} layers (t_layer={t_layer*1e3:.1f} ms, t_head={t_head*1e3:.1f} ms)")
        return self.batch / t_full, desc, times[1] + times[2]


def cpu_port_decode(batch: int, ctx: int, layers_full: int, n_rep: int = 1):
    port = CpuPortStep(batch, ctx, layers_full)
    best, desc, secs = None, "", 0.0
    for _ in range(n_rep):
        tps, desc, t = port.sample()
        best = tps if best is None else max(best, tps)
        secs += t
    return best, desc, secs


def engine_ttft(gpus, layout: str, quick: bool = False, qps: float = None, clock: str = "device"):
    """Turn-2+ TTFT / TPOT, PD (x=0) vs PPD (x=1), through the host C++ engine
    on the DEVICE clock: every prefill chunk, decode iteration and P->D KV hop
    runs on the GPUs listed (node i -> gpus[i]); each node's clock advances by
    the CUDA-event time of its own work. 1P_1D uses the BASELINE configs[2]
    trace (4 turns of 1536 in / 512 out); the 8-node layouts use configs[3]
    (2048 then 2x1024 in, 128 out, high load)."""
    from paper_2603_13358_b200 import engine as E
    if layout in ("1P_1D", "1R"):
        # BASELINE configs[2]: 4 turns, +2048 tokens of context per turn (1536 in, 512 out)
        wl = cfg2_workload(qps or 1.0, quick)
    else:
        wl = {"id": "cfg4", "turn1": [2048, 128], "turn2plus": [1024, 128], "num_turns": 3,
              "qps": 8.0, "duration_s": 4.0 if quick else 8.0}
    distinct = len(set(gpus)) == len(gpus)
    out = {"cluster": layout, "workload": wl, "model": "llama-3-8b-shape", "gpus": gpus, "clock": clock,
           "placement": ("one node per GPU" if distinct else "nodes share GPU %s" % sorted(set(gpus)))
           + ("; device clock = per-node CUDA-event durations" if clock == "device" else
              "; realtime = wall clock, one worker thread per node, asynchronous NVLink KV hops")}
    for x in (0.0, 1.0):
        job = {"cluster": layout, "x": x, "clock": clock, "seed": 3, "workload": wl,
               "device": {"model": "llama8b", "weight_seed": SEED, "token_seed": 3, "gpus": gpus,
                          "kv_blocks_per_node": 0, "prefill_chunk": 2048, "record_tokens": False}}
        t0 = time.perf_counter()
        r = E.run(job)
        agg = r["aggregate"]
        ms = lambda v: None if v is None else v * 1e3
        out[f"x{int(x)}"] = {"ttft_t2_p50_ms": ms(agg["ttft_t2_p50"]), "ttft_t2_p99_ms": ms(agg["ttft_t2_p99"]),
                             "ttft_t2_mean_ms": ms(agg["ttft_t2_mean"]), "tpot_mean_ms": ms(agg["tpot_mean"]),
                             "tpot_p50_ms": ms(agg["tpot_p50"]), "success_rate": agg["success_rate"],
                             "decode_tok_s": agg["tps"],
                             "link_transfers": r["link_transfers"], "link_gb": r["link_bytes"] / 1e9,
                             "link_bytes": r["link_bytes"],
                             "kv_transfer_gbs": r["device"]["kv_transfer"]["gbs"],
                             "kv_hop_ms_p50": r["device"]["kv_transfer"]["hop_ms_p50"],
                             "kv_blocks_in_use_at_end": r["device"]["kv_lifecycle"]["blocks_in_use_at_end"],
                             "wall_s": time.perf_counter() - t0}
    p0, p1 = out["x0"]["ttft_t2_p50_ms"], out["x1"]["ttft_t2_p50_ms"]
    if p0 and p1:
        out["ttft_t2_p50_reduction"] = 1.0 - p1 / p0
    return out


def qwen_long_decode(local_rank, B=16, ctx0=16384, K=5, W=3):
    """BASELINE configs[4]'s model on one GPU: Qwen2.5-32B-shape (GQA 40/8,
    QKV bias, random-init bf16, 65.5 GB of weights) decoding B sequences at a
    16k-token context (the 'large' router class). KV filled with random bf16
    (the step reads every byte regardless). Device time, CUDA events."""
    import paper_2603_13358_b200 as ppd
    cfg = ppd.qwen32b_cfg()
    BT = 16
    bps = (ctx0 + W + K + BT) // BT + 1
    dev = ppd.Device(local_rank, cfg, max_step_tokens=256, max_step_seqs=max(B, 8))
    try:
        dev.load_random_weights(SEED)
        dev.kv_pool_init(B * bps)
        ptr, nbytes = dev.kv_pool_ptr()
        ppd.check(ppd.lib().ppd_op_fill_random(ptr, nbytes // 2, SEED, 99, 0, None))
        bts = np.arange(B * bps, dtype=np.int32).reshape(B, bps)
        ctx = np.full(B, ctx0, dtype=np.int32)
        tok = np.random.default_rng(SEED).integers(0, cfg.vocab, B).astype(np.int32)
        ms = []
        for i in range(W + K):
            r = dev.step([1] * B, ctx, tok, bts)
            tok = r.tokens
            ctx += 1
            if i >= W:
                ms.append(r.ms)
        t = float(np.mean(ms))
        kv_bytes = float(np.sum(ctx - 1)) * 262144
        w_bytes = 65.5e9
        pk, _ = peaks()
        return {"model": "qwen2.5-32b-shape (random init, QKV bias, GQA 40/8)", "batch": B, "ctx": ctx0,
                "tpot_ms": t, "tok_s": B / (t * 1e-3), "step_bytes": kv_bytes + w_bytes,
                "step_hbm_gbs": (kv_bytes + w_bytes) / (t * 1e-3) / 1e9,
                "step_hbm_frac": (kv_bytes + w_bytes) / (t * 1e-3) / 1e9 / pk["hbm_gbs"], "steps": K}
    finally:
        dev.close()


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cfg2_workload(qps: float, quick: bool = False) -> dict:
    """BASELINE configs[2]: 4 turns of 1536 in / 512 out (+2048 context per turn)."""
    return {"id": "cfg3", "turn1": [1536, 512], "turn2plus": [1536, 512], "num_turns": 4,
            "qps": qps, "duration_s": 4.0 if quick else 12.0}


def reference_des(cluster: str, wl: dict, seed: int, calib: dict) -> dict:
    """The UNMODIFIED reference (oracle/_ref/ref_tool = /root/reference/proj/src
    built by oracle/Makefile) simulating the identical trace: its simulated
    turn-2+ TTFT / TPOT, link bytes and the DES wall time on this host."""
    from oracle import oracle as O
    out = {}
    for x in (0.0, 1.0):
        r = O.ref_tool({"op": "simulate", "cluster": cluster, "x": x, "workload": wl, "seed": seed, **calib})
        a = r["aggregate"]
        ms = lambda v: None if v is None else v * 1e3
        # the reference aggregates mean / p99 only; p50 by its own nearest-rank rule (metrics.cpp:43-60)
        recs = [json.loads(l) for l in r["records_jsonl"].splitlines()[1:]]
        t2 = sorted(v["first_token"] - v["arrival"] for v in recs
                    if v["turn_index"] >= 2 and v.get("first_token") is not None and v["status"] == "completed")
        p50 = t2[max(0, int(np.ceil(0.5 * len(t2))) - 1)] if t2 else None
        out[f"x{int(x)}"] = {"ttft_t2_p50_ms": ms(p50), "ttft_t2_p99_ms": ms(a.get("ttft_t2_p99")),
                             "tpot_mean_ms": ms(a.get("tpot_mean")), "decode_tok_s": a.get("tps"),
                             "link_transfers": r["link_transfers"], "link_bytes": r["link_bytes"],
                             "des_wall_s": r["wall_s"], "calib_hash": r["calib_hash"]}
    p0, p1 = out["x0"]["ttft_t2_p50_ms"], out["x1"]["ttft_t2_p50_ms"]
    if p0 and p1:
        out["ttft_t2_p50_reduction"] = 1.0 - p1 / p0
    return out


def reference_sweep() -> dict:
    """the reference's default sweep plan (9,180 DES cells) with
    parallelism = nproc, run by the UNMODIFIED reference (oracle/_ref/ref_tool,
    sweep.cpp run_sweep) and by the engine's own sweep (engine/sweep) on the
    same plan: wall times and whether the two cell CSVs are byte-identical."""
    import time as _t
    from oracle import oracle as O
    from paper_2603_13358_b200 import engine as E
    plan = json.loads(E.run({"op": "plan_default"})["plan_json"])
    par = os.cpu_count() or 1
    t0 = _t.perf_counter()
    r = O.ref_tool({"op": "sweep", "plan": plan, "parallelism": par})
    t_ref = _t.perf_counter() - t0
    t0 = _t.perf_counter()
    m = E.run({"op": "sweep", "plan": plan, "parallelism": par})
    t_ours = _t.perf_counter() - t0
    return {"plan": "reference default plan", "cells": len(r["cells"]), "parallelism": par,
            "host_cpu_model": cpu_model(), "reference_wall_s": t_ref, "engine_wall_s": t_ours,
            "plan_hash": r["plan_hash"], "csv_identical": r["csv"] == m["csv"],
            "winner_cells": r["winner"]["cells"]}


def device_calibration(dev, cfg, inter: dict, B: int, ctx, tok, bts, cal_bt, link_gbs: float) -> dict:
    """CalibrationTable coefficients fitted from B200 measurements of this run
    (ppd::cost::fit_from_measurements through the engine's fit_calibration op):
    decode steps at 4 batch sizes, full prefills at 3 lengths, appends of 1536
    tokens at 3 cached lengths, the interference sweep's multipliers and the
    measured KV-hop bandwidth (reference schema: costmodel.cpp:197-316)."""
    from paper_2603_13358_b200 import engine as E
    rng = np.random.default_rng(SEED + 7)
    def med(f, n=3):
        f()
        f()  # first call of a shape runs eagerly, the second captures its CUDA graph
        return float(np.median([f() for _ in range(n)]))
    samples = {"decode": [], "full": [], "append": [], "interference": [],
               "kv_bytes_per_token": 131072.0, "link_bandwidth": link_gbs * 1e9}
    for b in (8, 50, 100, B):
        t = med(lambda: dev.step([1] * b, ctx[:b], tok[:b], bts[:b]).ms)
        samples["decode"].append([b, t * 1e-3])
    for n in (1024, 2048, 4096):
        toks = rng.integers(0, cfg.vocab, n).astype(np.int32)
        t = med(lambda: dev.step([n], [0], toks, cal_bt).ms, 2)
        samples["full"].append([n, t * 1e-3])
    for n in (2048, 4096, 6144):
        toks = rng.integers(0, cfg.vocab, 1536).astype(np.int32)
        t = med(lambda: dev.step([1536], [n], toks, cal_bt).ms, 2)
        samples["append"].append([1536, n, t * 1e-3])
    for conc in (1, 4):
        c = inter[f"conc{conc}"]
        samples["interference"].append({"kind": "full", "prefill_tokens": 1024, "concurrent_prefills": conc,
                                        "decode_batch": B, "tpot_multiplier": c["mult_full"]})
        samples["interference"].append({"kind": "append", "prefill_tokens": 1024, "concurrent_prefills": conc,
                                        "decode_batch": B, "tpot_multiplier": c["mult_append"]})
    fit = E.run({"op": "fit_calibration", "samples": samples})
    return {"samples": samples, "calib_json": fit["calib_json"], "hash": fit["hash"]}


def nvlink_probe(world: int) -> dict:
    """NVLink roofline (N > 1): GPU0 -> GPU1 copy bandwidth, best of 5 x 1 GiB,
    through the copy engines and through an SM pull kernel; then the K7 KV-hop
    kernel (ppd_kv_copy) between two Llama-3-8B-shape pools on GPU 0 and GPU 1
    at 1536 and 8192 tokens, as a fraction of the best measured peak."""
    import paper_2603_13358_b200 as ppd
    g0, g1 = gpu_of(0), gpu_of(1)
    out = {"pair": [g0, g1], "dry_run_same_gpu": SAME_GPU}
    out["ce_gbs"] = ppd.p2p_bandwidth(g0, g1, 1 << 30, 5, 0)
    out["sm_pull_gbs"] = ppd.p2p_bandwidth(g0, g1, 1 << 30, 5, 1)
    out["hbm_copy_gbs_same_gpu"] = ppd.p2p_bandwidth(g0, g0, 1 << 30, 5, 1)
    peak = max(out["ce_gbs"], out["sm_pull_gbs"])
    out["peak_gbs"] = peak
    out["peak_kind"] = "measured (best of copy-engine / SM-pull probe)"
    out["nominal_gbs"] = 900.0
    cfg = ppd.llama8b_cfg()
    devs = [ppd.Device(g, cfg, max_step_tokens=256, max_step_seqs=8) for g in (g0, g1)]
    try:
        for d in devs:
            d.kv_pool_init(1024)
        kvb = ppd.kv_block_bytes(cfg) / 16
        for n in (1536, 8192):
            nb = (n + 15) // 16
            src = np.arange(nb, dtype=np.int32)
            dst = np.arange(512 - nb // 2, 512 - nb // 2 + nb, dtype=np.int32) % 1024
            ms = min(ppd.kv_copy(devs[0], devs[1], src, dst, 0, n) for _ in range(5))
            gbs = n * kvb / (ms * 1e-3) / 1e9
            out[f"k7_{n}_tokens"] = {"ms": ms, "gbs": gbs, "frac_of_peak": gbs / peak if peak else None,
                                     "frac_of_nominal": gbs / 900.0}
    finally:
        for d in devs:
            d.close()
    return out


_HOST_GROUP = None


def host_group():
    """A gloo group over the same ranks, created by every rank right after init."""
    return _HOST_GROUP


def bench_config(B: int, ctx0: int, world: int) -> dict:
    return {
        "workload": f"Llama-3-8B-shape decode step, B={B} requests at ctx {ctx0}+, 1 colocated node per GPU "
                    "(BASELINE configs[1]); interference sweep beside it",
        "model": "llama-3-8b-shape (random init)",
        "global_batch": B * world,
        "seq_len": ctx0,
        "parallelism": "replicas (one node per GPU, no collective in the decode step)",
        "l2_policy": f"inputs larger than L2: {B * ctx0 * 131072 / 1e9:.1f} GB KV + 16.06 GB weights read per step",
    }


# ----------------------------------------------------------------- our arm
def run_ours(args, rank, world, local_rank):
    import torch
    import paper_2603_13358_b200 as ppd

    local_rank = gpu_of(local_rank)
    torch.cuda.set_device(local_rank)
    cfg = ppd.llama8b_cfg()
    B, ctx0 = args.batch, args.ctx
    K, W = args.steps, args.warmup
    BT = 16
    max_ctx = ctx0 + W + K + 16
    bps = (max_ctx + BT - 1) // BT
    n_inter_blocks = 4 * 64 + 4 * 64 + 8
    n_cal_blocks = (6144 + 1536) // 16 + 8  # calibration prefills / appends
    dev = ppd.Device(local_rank, cfg, max_step_tokens=max(4096, B + 4 * 1024), max_step_seqs=max(B + 8, 256))
    dev.load_random_weights(SEED)
    dev.kv_pool_init(B * bps + n_inter_blocks + n_cal_blocks)
    bts = np.arange(B * bps, dtype=np.int32).reshape(B, bps)
    rng = np.random.default_rng(SEED + rank)

    # ---- prefill the B contexts (4 sequences of ctx0 tokens per step) ----
    t0 = time.perf_counter()
    last = np.zeros(B, dtype=np.int32)
    if args.fill_kv == "random":
        ptr, nbytes = dev.kv_pool_ptr()
        ppd.check(ppd.lib().ppd_op_fill_random(ptr, nbytes // 2, SEED, 99, 0, None))
        last[:] = rng.integers(0, cfg.vocab, B)
    else:
        per = max(1, 4096 // ctx0)
        for s0 in range(0, B, per):
            idx = list(range(s0, min(B, s0 + per)))
            toks = rng.integers(0, cfg.vocab, ctx0 * len(idx)).astype(np.int32)
            r = dev.step([ctx0] * len(idx), [0] * len(idx), toks, bts[idx])
            last[idx] = r.tokens
    prefill_s = time.perf_counter() - t0

    ctx = np.full(B, ctx0, dtype=np.int32)
    tok = last.copy()
    for _ in range(W):
        tok = dev.step([1] * B, ctx, tok, bts).tokens
        ctx += 1

    # ---- timed region: K decode steps ----
    dist = world > 1
    if dist:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    dev.reset_stats()
    ncu = bool(os.environ.get("PPD_NCU"))
    if ncu:
        torch.cuda.profiler.start()
    with ClockSampler(local_rank) as clk:
        t0 = time.perf_counter()
        step_ms = []
        for _ in range(K):
            r = dev.step([1] * B, ctx, tok, bts)
            tok = r.tokens
            step_ms.append(r.ms)
            ctx += 1
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    if ncu:
        torch.cuda.profiler.stop()
        dev.close()
        return
    if dist:
        torch.distributed.barrier()
    st = dev.stats()
    dev_ms = float(np.sum(step_ms))
    h2d_bytes = 4 * (B + 1 + B + B + B * bps + B + B + B) + 48 * B * 2
    times = torch.tensor([dev_ms, wall * 1e3], dtype=torch.float64, device="cpu" if SAME_GPU else "cuda")
    if dist:
        torch.distributed.all_reduce(times, op=torch.distributed.ReduceOp.MAX)
    dev_ms_max, wall_ms_max = times.tolist()

    # ---- profiled pass: per-kernel-class device time (roofline) ----
    dev.set_profiling(True)
    dev.reset_stats()
    for _ in range(3):
        tok = dev.step([1] * B, ctx, tok, bts).tokens
        ctx += 1
    prof = dev.stats()
    dev.set_profiling(False)

    # ---- interference sweep (configs[1]): prefills riding in the decode step ----
    inter = {}
    base_blk = B * bps
    ib = lambda i: np.arange(base_blk + 64 * i, base_blk + 64 * (i + 1), dtype=np.int32)
    # cached contexts for the append sequences: n = 1024 - m tokens each
    m_app = args.append_new
    for i in range(4):
        dev.step([1024 - m_app], [0], rng.integers(0, cfg.vocab, 1024 - m_app), ib(4 + i))

    def timed(extra_q, extra_ctx, extra_bt, n=5, warm=2):
        # the first call of a step shape runs eagerly and the second captures its CUDA
        # graph (device.cu run_step); both are warm-up, the median is over graph replays
        q = [1] * B + extra_q
        c = list(ctx) + extra_ctx
        bt = np.zeros((B + len(extra_q), bps + 64), dtype=np.int32)
        bt[:B, :bps] = bts
        for j, e in enumerate(extra_bt):
            bt[B + j, :64] = e
        want = [1] * B + [0] * len(extra_q)
        ms = []
        for i in range(warm + n):
            toks = np.concatenate([tok, rng.integers(0, cfg.vocab, int(np.sum(extra_q)))]).astype(np.int32)
            t = dev.step(q, c, toks, bt, want).ms
            if i >= warm:
                ms.append(t)
        return float(np.median(ms))

    alone = timed([], [], [])
    for conc in (1, 4):
        full = timed([1024] * conc, [0] * conc, [ib(i) for i in range(conc)])
        app = timed([m_app] * conc, [1024 - m_app] * conc, [ib(4 + i) for i in range(conc)])
        inter[f"conc{conc}"] = {"tpot_ms_full_1024": full, "tpot_ms_append_1024": app,
                                "mult_full": full / alone, "mult_append": app / alone}
    inter["tpot_ms_alone"] = alone
    inter["append_new_tokens"] = m_app
    inter["reference_anchor_mult"] = {"full_1024_b200": 1.48, "append_1024_b200": 1.02,
                                      "full_1024_conc4": 1.57, "append_1024_conc4": 1.21}

    def guarded(fn, *a, **k):
        # a failing side measurement is reported in the line, never kills it
        try:
            return fn(*a, **k)
        except Exception as e:  # noqa: BLE001
            return {"error": f"{type(e).__name__}: {e}"}

    cal = None
    if rank == 0 and not args.quick:
        cal_bt = np.arange(B * bps + n_inter_blocks, B * bps + n_inter_blocks + n_cal_blocks, dtype=np.int32)
        cal = guarded(device_calibration, dev, cfg, inter, B, ctx, tok, bts, cal_bt, 0.0)
    dev.close()
    if rank != 0:
        if world > 1:
            # rank 0 drives all GPUs for the engine runs: wait on the CPU (gloo), since an
            # NCCL barrier would spin a kernel on this GPU and time-slice against rank 0's work
            torch.distributed.barrier(group=host_group())
        return

    qwen = None
    if not args.no_qwen and not args.quick:
        qwen = guarded(qwen_long_decode, local_rank)
    nvlink = guarded(nvlink_probe, world) if world > 1 else None
    ttft = None
    if not args.no_engine:
        from paper_2603_13358_b200 import dist as D
        if world == 1:
            # configs[2] at two loads of the SURVEY §8d C3 QPS sweep
            ttft = [guarded(engine_ttft, [local_rank, local_rank], "1P_1D", quick=args.quick, qps=q)
                    for q in ((1.0,) if args.quick else (1.0, 2.0))]
        else:
            # one node per GPU, wall clock: steps of different nodes run concurrently and
            # every KV hop overlaps its destination's decode steps
            ttft = [guarded(engine_ttft, [gpu_of(g) for g in D.layout_gpus(lay, world)], lay, quick=args.quick,
                            clock="realtime")
                    for lay in D.node_layouts(world)]
            if isinstance(nvlink, dict) and nvlink.get("peak_gbs"):
                for t in ttft:
                    for x in ("x0", "x1"):
                        if isinstance(t, dict) and x in t and t[x].get("kv_transfer_gbs"):
                            t[x]["kv_transfer_frac_of_nvlink_peak"] = t[x]["kv_transfer_gbs"] / nvlink["peak_gbs"]
    # the reference DES on the identical traces, default and device-fitted calibration
    des = None
    if not args.no_cpu and ttft:
        des = []
        link_gbs = 0.0
        for t in ttft:
            if isinstance(t, dict) and "x0" in t and t["x0"].get("kv_transfer_gbs"):
                link_gbs = max(link_gbs, t["x0"]["kv_transfer_gbs"])
        if isinstance(cal, dict) and "samples" in cal and link_gbs > 0:
            from paper_2603_13358_b200 import engine as E
            cal["samples"]["link_bandwidth"] = link_gbs * 1e9
            fit = guarded(E.run, {"op": "fit_calibration", "samples": cal["samples"]})
            if isinstance(fit, dict) and "calib_json" in fit:
                cal["calib_json"], cal["hash"] = fit["calib_json"], fit["hash"]
        for t in ttft:
            if not (isinstance(t, dict) and "workload" in t):
                continue
            row = {"cluster": t["cluster"], "qps": t["workload"]["qps"],
                   "default_calibration_llama8b_kv": guarded(reference_des, t["cluster"], t["workload"], 3,
                                                             {"calib_overrides": {"kv_bytes_per_token": 131072}})}
            if isinstance(cal, dict) and "calib_json" in cal:
                row["device_fitted_calibration"] = guarded(reference_des, t["cluster"], t["workload"], 3,
                                                           {"calib_json": cal["calib_json"]})
            d0 = row["default_calibration_llama8b_kv"]
            if isinstance(d0, dict) and "x0" in d0:
                row["link_bytes_equal_device_run"] = all(
                    d0[x]["link_bytes"] == t[x]["link_bytes"] for x in ("x0", "x1") if x in t)
            des.append(row)

    pk, pk_kind = peaks()
    traffic = None  # dram read+write per launch of the same kernel/config, from the committed ncu capture
    try:
        prof_ncu = json.load(open(os.path.join(REPO, "profiles", "ncu_r02l_kernels.json")))
        k0 = prof_ncu["decode_attention_B200_ctx1024_layer0"][0]
        if B == 200 and ctx0 == 1024:
            num = lambda v: float(str(v).split()[0])  # "854.9 Mbyte" or "854.9" (MB)
            traffic = (num(k0["dram__bytes_read.sum"]) + num(k0["dram__bytes_write.sum"])) * 1e6
    except Exception:
        pass
    attn_gbs = prof["attn_bytes"] / (prof["attn_ms"] * 1e-3) / 1e9 if prof["attn_ms"] > 0 else None
    total_prof_ms = prof["step_ms"]
    step_bytes_kv = float(np.sum(ctx)) * 131072
    value = B * K * world / (dev_ms_max * 1e-3)
    e2e_value = B * K * world / (wall_ms_max * 1e-3)

    cpu = None
    if not args.no_cpu:
        nthr = cpu_threads()
        tps, sample, secs = cpu_port_decode(args.cpu_batch, ctx0, cfg.n_layers)
        cpu = {"value": tps, "unit": "tok/s", "cores": nthr, "kind": "port", "sample": sample,
               "wall_s": secs, "host_cpu_model": cpu_model(), "host_nproc": os.cpu_count(),
               "reference_des": des}
        try:
            cpu["reference_sweep"] = reference_sweep()
        except Exception as e:  # noqa: BLE001
            cpu["reference_sweep"] = {"error": f"{type(e).__name__}: {e}"}

    line = {
        "metric": METRIC,
        "value": value,
        "unit": "tok/s",
        "n_gpus": world,
        "steps": K,
        "warmup": W,
        "ms_per_step": dev_ms_max / K,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic token ids, random-init bf16 weights (counter hash, std 0.02)",
        "config": bench_config(B, ctx0, world),
        "tpot_ms": dev_ms_max / K,
        "interference": inter,
        "ttft_pd_vs_ppd": ttft,
        "nvlink": nvlink,
        "device_calibration": ({k: v for k, v in cal.items() if k != "calib_json"} if isinstance(cal, dict) else cal),
        "qwen32b_long_decode": qwen,
        "roofline": {
            "kernel": "decode_attention_kernel (K1, balanced persistent paged decode attention)",
            "bound": "hbm",
            "achieved": attn_gbs,
            "peak": pk["hbm_gbs"],
            "peak_kind": pk_kind,
            "unit": "GB/s",
            "frac": (attn_gbs / pk["hbm_gbs"]) if attn_gbs else None,
            "traffic": traffic,
            "traffic_source": "profiles/ncu_r02l_kernels.json (ncu --set full, dram__bytes_read+write per launch)",
            "algorithmic_bytes_per_launch": prof["attn_bytes"] / max(prof["attn_launches"], 1),
            "attn_share_of_step": prof["attn_ms"] / total_prof_ms if total_prof_ms else None,
            "gemm_share_of_step": prof["gemm_ms"] / total_prof_ms if total_prof_ms else None,
        },
        "step_hbm": {
            "bytes_per_step": step_bytes_kv + 16.06e9,
            "achieved_gbs": (step_bytes_kv + 16.06e9) / (dev_ms_max / K * 1e-3) / 1e9,
        },
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "tok/s", "h2d_bytes_per_step": h2d_bytes,
                "d2h_bytes_per_step": 4 * B},
        "gpu_launches": int(st["own_launches"]),
        "lib_launches": int(st["lib_launches"]),
        "clocks": clk.summary(),
        "prefill_setup_s": prefill_s,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier(group=host_group())


def run_reference(args, rank, world):
    """The reference arm: the reference prices this step analytically
    (costmodel.cpp:372-379) and computes no tokens, so its CPU implementation
    of the step is the oracle port (kind "port"), on all host threads, W + K
    bounded samples (each ~1-2 s). The unmodified reference DES is run beside
    it on the configs[2] trace (kind "reference")."""
    if rank != 0:
        return
    nthr = cpu_threads()
    port = CpuPortStep(args.cpu_batch, args.ctx, 32)
    for _ in range(args.warmup):
        port.sample()
    vals, sample, t_all = [], "", 0.0
    for _ in range(args.steps):
        tps, sample, secs = port.sample()
        vals.append(tps)
        t_all += secs
    v = float(np.median(vals))
    des = None
    try:
        des = reference_des("1P_1D", cfg2_workload(1.0), 3, {"calib_overrides": {"kv_bytes_per_token": 131072}})
    except Exception as e:  # noqa: BLE001
        des = {"error": f"{type(e).__name__}: {e}"}
    try:
        sweep = reference_sweep()
    except Exception as e:  # noqa: BLE001
        sweep = {"error": f"{type(e).__name__}: {e}"}
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": v,
        "unit": "tok/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": float(np.median([args.cpu_batch / x for x in vals])) * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32 (bf16 storage)",
        "data": "synthetic token ids, random-init bf16 weights (counter hash, std 0.02)",
        "config": bench_config(args.batch, args.ctx, world),
        "cpu_baseline": {"value": v, "unit": "tok/s", "cores": nthr, "kind": "port", "sample": sample,
                         "host_cpu_model": cpu_model(), "samples_s": t_all},
        "reference_des": {"kind": "reference", "what": "unmodified reference DES (oracle/_ref/ref_tool) on the "
                          "configs[2] trace, 1P_1D, seed 3, QPS 1, default calibration with Llama-3-8B KV bytes",
                          "result": des},
        "reference_sweep": sweep,
        "e2e": {"value": v, "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "the reference (/root/reference/proj) prices this step analytically "
                "(costmodel.cpp:372-379) and computes no tokens; its CPU arm is the oracle port",
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=200)
    ap.add_argument("--ctx", type=int, default=1024)
    ap.add_argument("--append-new", type=int, default=128)
    ap.add_argument("--cpu-batch", type=int, default=200)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--fill-kv", default="prefill", choices=["prefill", "random"])
    ap.add_argument("--no-engine", action="store_true")
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--no-qwen", action="store_true")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        torch.cuda.set_device(gpu_of(local_rank))
        import datetime
        torch.distributed.init_process_group("gloo" if SAME_GPU else "nccl", timeout=datetime.timedelta(minutes=30))
        global _HOST_GROUP
        _HOST_GROUP = torch.distributed.new_group(backend="gloo", timeout=datetime.timedelta(minutes=60))
    run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
