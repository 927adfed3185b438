"""bench.py -- MarginGate decode throughput on B200 (BASELINE.json configs[1]).

Workload (N=1): Llama-3.1-8B-shaped random-init decoder (DESIGN.md 3.1
weights, seed 42), batch 64 per GPU, MATH500-shaped request (prompt 128 /
decode 512): the K timed steps are the LAST K steps of that
decode (contexts up to 640), past the verifier's 512-key attention split, where
the batch-64 fast plan and the verifier's pinned plan differ
and MarginGate's gate has real work (calibrated tau100 > 0).  One bench
"step" = one mg_decode_step = one pass of the whole hot path (SURVEY 8(a)
rows a1-a11) over the batch.

Three arms, each from the same deterministic prefill, W warm-up + K timed
steps: tau = 0 (pure BF16, r_verify = 0), tau = tau_op (MarginGate, the
headline `value`), tau = +inf (always-on verification, LLM-42 analog,
PAPER.md:215).  Reported: decode tok/s (whole job), the latency increments
inc = T/T_bf16 - 1 and their ratio inc_AO / inc_MG, trigger
% (r_verify) and determinism % (protected rows whose MarginGate sequence is
bit-identical to the always-on run, which the GPU tests prove equal to the
batch-1 reference).

N > 1 (torchrun): requests are sharded, every rank decodes its own batch of
64; the only collective is an NCCL all-reduce of the int64 stats vector and
max over ranks of the device time.  scaling = weak.

--impl reference: the CPU oracle, as it stands, on the same workload, one
bounded sample (one row of the batch) per step.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode tok/s + latency increment vs always-on verify; trigger %; determinism %"
# calibration prompts (tau100) come from seeds CALIB_SEED + i, disjoint from the
# evaluation seeds 7 + i of every rank at any world size
CALIB_SEED = 10 ** 6


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md recipe)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.nv = None
        self.err = None
        self.stop_ev = threading.Event()

    def start(self):
        """Sample the SM clock and the throttle reasons every 5 ms through NVML
        (nvidia-smi's 200 ms floor would give one sample of a short region)."""
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.h = h
            self._sample(h)  # one synchronous sample at the start of the region
            self.t = threading.Thread(target=self._nvml, args=(h,), daemon=True)
            self.t.start()
            return
        except Exception:
            self.nv = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _sample(self, h):
        nv = self.nv
        bits = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                "sw_power_cap": 0x4}
        reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        try:
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        except Exception as e:  # noqa: BLE001
            self.err = repr(e)
            return
        try:
            r = reasons(h)
        except Exception as e:  # noqa: BLE001
            self.err = repr(e)
            r = 0
        self.rows.append(["", str(sm), str(mx), "", "", *["Active" if r & bits[k] else "Not Active"
                                                          for k in ("hw_slowdown", "hw_thermal_slowdown",
                                                                    "sw_thermal_slowdown", "sw_power_cap")]])

    def _nvml(self, h):
        while not self.stop_ev.is_set():
            self._sample(h)
            time.sleep(0.005)

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.nv is not None:
            self._sample(self.h)  # and one at its end (the sampler thread may not have run)
        self.stop_ev.set()
        if self.nv is not None:
            self.t.join(timeout=2)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        sm = [float(r[1]) for r in self.rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 8 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            if len(r) > 8:
                for n, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(n)
        out = {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
               "reasons": sorted(reasons), "samples": len(sm), "source": "nvml 5 ms" if self.nv else "nvidia-smi"}
        if getattr(self, "err", None):
            out["error"] = self.err
        return out


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def run_gpu(args):
    import torch
    import torch.distributed as dist

    from paper_2605_30218_b200 import inputs, metrics, sharding
    from paper_2605_30218_b200.engine import Engine

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    if ws > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    shp = inputs.shape(args.model)
    B, K, W = args.batch, args.steps, args.warmup
    prompt_len, decode_len = inputs.WORKLOADS[args.workload]
    ctx0 = max(prompt_len, prompt_len + decode_len - W - K)   # the timed steps end the decode
    max_seq = ctx0 + W + K + 2
    eng = Engine(shp, max_batch=B, max_slots=B, max_seq=max_seq, page_size=64)
    # requests of this rank: global ids rank*B .. rank*B + B-1 (request i -> rank i // B)
    prompts = inputs.prompts(B, ctx0, shp["vocab"], seed=7 + sharding.rank_requests(rank, ws, B)[0])
    if ws > 1:
        # cross-rank determinism probe: row 0 of every rank decodes
        # global request 0 (protected), each time inside a different batch
        prompts[0] = inputs.prompts(1, ctx0, shp["vocab"], seed=7)[0]
    out = torch.empty(B, dtype=torch.int32, device="cuda")
    kind = torch.empty(B, dtype=torch.uint8, device="cuda")
    stream = eng.stream
    keys = ["steps", "rows", "protected_rows", "triggers", "verified", "repairs", "verifier_launches",
            "catchup_tokens"]

    def run_arm(tau, prot, timing=False, clocks=None, pipelined=False, fused=False, arm_prompts=None):
        """Fresh deterministic prefill, W warm-up steps, K timed steps (CUDA events
        on the engine's stream, barrier + synchronize on both sides).
        pipelined: MG_VERIFY_PIPELINED (include/mg.h) -- a gated row's
        verifier rides on its next step; tokens = emitted minus replaced (kind 4)."""
        for i in range(B):
            try:
                eng.release(i)
            except Exception:
                pass
        eng.set_policy(verify_mode=1 if pipelined else (2 if fused else 0))
        ps = arm_prompts or prompts
        first = [eng.prefill(i, p) for i, p in enumerate(ps)]
        s0 = eng.stats()
        toks, kinds_w = [], []
        for _ in range(W):
            eng.step(list(range(B)), prot, tau, out, kind)
            toks.append(out.cpu().numpy().copy())
            kinds_w.append(kind.cpu().numpy().copy())
        eng.set_timing(timing)
        if clocks:
            clocks.start()
        l0 = eng.launches()
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        outs = torch.empty((K, B), dtype=torch.int32, device="cuda")
        kinds = torch.empty((K, B), dtype=torch.uint8, device="cuda")
        prof = clocks is not None and os.environ.get("MG_PROFILE_TIMED") == "1"  # ncu --profile-from-start off
        if prof:
            torch.cuda.profiler.start()
        e0.record(stream)
        for k in range(K):
            eng.step(list(range(B)), prot, tau, outs[k], kinds[k])
        e1.record(stream)
        if prof:
            torch.cuda.synchronize()
            torch.cuda.profiler.stop()
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        r = dict(ms=e0.elapsed_time(e1), launches=eng.launches() - l0)
        if timing:
            r["tim"] = eng.timing()
            eng.set_timing(False)
            r["tim"]["floor_us"] = _launch_floor(eng)
        if clocks:
            r["clk"] = clocks.stop()
        s1 = eng.stats()
        kt = kinds.cpu().numpy()
        toks += list(outs.cpu().numpy())
        kall = kinds_w + list(kt)
        seqs = [[first[b]] for b in range(B)]
        for t, kk in zip(toks, kall):
            for b in range(B):
                if pipelined and kk[b] == 4:
                    seqs[b][-1] = int(t[b])
                else:
                    seqs[b].append(int(t[b]))
        if pipelined:  # resolve the last tentative tokens (untimed)
            pos, last, _ = eng.verify_window(list(range(B)))
            for b in range(B):
                n = int(pos[b]) - len(ps[b]) + 1
                del seqs[b][n:]
                seqs[b][-1] = int(last[b])
            eng.set_policy(verify_mode=0)
        if fused:
            eng.set_policy(verify_mode=0)
        r["seqs"] = seqs
        r["tokens"] = int(B * K - (kt == 4).sum()) if pipelined else B * K
        r["stats"] = {k: s1[k] - s0[k] for k in keys}
        return r

    prot_one, prot_all = inputs.protected_mask(B, "one"), inputs.protected_mask(B, "all")
    head = prot_one if args.protected == "one" else prot_all
    # operating threshold: the paper's protocol -- tau100
    # calibrated on disjoint seeds (10^6 + i) -- unless --tau fixes it; ranks
    # agree on the largest (most conservative) value
    calib = None
    tau = args.tau
    if tau is None:
        calib = calibrate(eng, inputs.prompts(B, ctx0, shp["vocab"], seed=CALIB_SEED + rank * B), W, K)
        t100 = calib["tau100"] if calib["tau100"] is not None else math.inf
        _, (tau,) = sharding.aggregate([], [t100], device="cuda")
    res = {"bf16": run_arm(0.0, None)}
    # the round-1 reference point: the BF16 step at the mid-decode context (~400)
    ctx_mid = prompt_len + decode_len // 2 - W
    res["bf16_mid"] = run_arm(0.0, None, arm_prompts=inputs.prompts(B, ctx_mid, shp["vocab"],
                                                                     seed=7 + sharding.rank_requests(rank, ws, B)[0]))
    res["mg"] = run_arm(tau, head, clocks=Clocks(local))
    res["ao"] = run_arm(math.inf, head)
    # pipelined verification (include/mg.h MG_VERIFY_PIPELINED): always-on with the
    # verifier riding on the next step's weight pass
    res["ao_pipe"] = run_arm(math.inf, head, pipelined=True)
    # fused same-step verification (MG_VERIFY_FUSED): synchronous semantics, one weight pass
    res["mg_fused"] = run_arm(tau, head, fused=True)
    res["ao_fused"] = run_arm(math.inf, head, fused=True)
    other = "all" if args.protected == "one" else "one"
    if not args.quick:
        po = prot_all if other == "all" else prot_one
        res["mg_other"] = run_arm(tau, po)
        res["ao_other"] = run_arm(math.inf, po)
        res["ao_pipe_other"] = run_arm(math.inf, po, pipelined=True)
        res["ao_fused_other"] = run_arm(math.inf, po, fused=True)
    # dominant-kernel timing pass: the fast path with CUDA events around every
    # GEMM / attention launch (events break the PDL overlap, so this pass is
    # separate from the timed arms; the per-launch durations are what ncu's
    # launch list shows, not the pipelined step)
    tim = run_arm(0.0, None, timing=True)["tim"]

    # ---- e2e: host buffers in and out through the C ABI every step (MarginGate arm)
    for i in range(B):
        eng.release(i)
    for i, p in enumerate(prompts):
        eng.prefill(i, p)
    for _ in range(W):
        eng.step(list(range(B)), head, tau, out, kind)
    h_out = torch.empty(B, dtype=torch.int32, pin_memory=True)
    h_kind = torch.empty(B, dtype=torch.uint8, pin_memory=True)
    h_slots = np.arange(B, dtype=np.int32)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(K):
        eng.step(h_slots, head, tau, out, kind)      # slots / mask copied H2D inside the call
        h_out.copy_(out, non_blocking=True)
        h_kind.copy_(kind, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)

    # ---- the paper's own protocol: batch 8, one
    # protected request, tau100 calibrated on disjoint seeds -- the regime
    # where the fast path's schedule really differs from the verifier's
    # ---- LLM-42-style windowed verify + rollback at the headline batch (NEXT-2;
    # K = --window, two windows), one and all rows protected, on an engine with
    # room for the extra positions (rank-local timing, like the paper arm)
    w64 = None
    if not args.quick and args.window > 0:
        eng.close()
        ew = Engine(shp, max_batch=B, max_slots=B, max_seq=ctx0 + W + 2 * args.window + 2, page_size=64)
        w64 = {}
        for pname, pm in (("one", prot_one), ("all", prot_all)):
            w64[pname] = _window_run(ew, prompts, pm, W, 2 * args.window, args.window)
        ew.close()
        eng = None

    # the whole MATH500-shaped decode at this batch (contexts 131..640 cross the
    # verifier's 512-key split): MarginGate's triggers, determinism and cost
    # where the fast path really differs from the verifier (rank-local)
    full = None
    if not args.quick and args.full_decode_arm:
        if eng is not None:
            eng.close()
            eng = None
        full = run_full_decode(args, pnames=("one", "all"))

    paper = None
    if not args.quick and args.paper_batch > 0:
        if eng is not None:
            eng.close()
        pb = args.paper_batch
        e8 = Engine(shp, max_batch=pb, max_slots=pb, max_seq=ctx0 + W + max(K, 2 * args.window) + 2, page_size=64)
        cal8 = calibrate(e8, inputs.prompts(pb, ctx0, shp["vocab"], seed=CALIB_SEED + rank * pb), 3, K)
        t8 = cal8["tau100"] if cal8["tau100"] is not None else math.inf
        _, (t8,) = sharding.aggregate([], [t8], device="cuda")
        ev8 = inputs.prompts(pb, ctx0, shp["vocab"], seed=7 + rank * pb)
        p1 = inputs.protected_mask(pb, "one")
        tp = cal8["tau_p"]  # 2 max eps: the argmax-bound threshold, conservative
        r8 = {n: _decode_run(e8, ev8, t, p1, W, K, timed=True)
              for n, t in (("bf16", 0.0), ("margingate", t8), ("margingate_tau_p", tp), ("always_on", math.inf))}
        # NEXT-3 repair-action ablation: token-only repair at tau100
        e8.set_policy(repair_action=1)
        r8["margingate_token_only"] = _decode_run(e8, ev8, t8, p1, W, K, timed=True)
        # NEXT-4 global batch-invariant baseline: every row on the pinned plan, tau = 0
        e8.set_policy(fast_schedule=1, repair_action=0)
        r8["batch_invariant"] = _decode_run(e8, ev8, 0.0, p1, W, K, timed=True)
        e8.set_policy(0, 0, 0)
        # pipelined verification (include/mg.h MG_VERIFY_PIPELINED)
        r8["margingate_pipelined"] = _decode_run(e8, ev8, t8, p1, W, K, timed=True, pipelined=True)
        r8["always_on_pipelined"] = _decode_run(e8, ev8, math.inf, p1, W, K, timed=True, pipelined=True)
        # fused same-step verification (MG_VERIFY_FUSED)
        r8["margingate_fused"] = _decode_run(e8, ev8, t8, p1, W, K, timed=True, fused=True)
        r8["always_on_fused"] = _decode_run(e8, ev8, math.inf, p1, W, K, timed=True, fused=True)
        # NEXT-2 LLM-42 windowed verify + rollback, K = 64, over 2 windows
        win = _window_run(e8, ev8, p1, W, 2 * args.window, args.window)
        e8.close()
        paper = {"batch": pb, "tau100": t8, "calibration": cal8, "r": r8, "window": win}

    # ---- aggregate over ranks (the only collectives: stats SUM, time MAX)
    def det(a, b, prot):
        return sum(1 for i in range(B) if prot[i] and res[a]["seqs"][i] == res[b]["seqs"][i]), int(prot.sum())

    arms = [a for a in ("bf16", "bf16_mid", "mg", "ao", "ao_pipe", "mg_fused", "ao_fused", "mg_other", "ao_other",
                        "ao_pipe_other", "ao_fused_other") if a in res]

    def det_prefix(a, b, prot):  # pipelined rows may be shorter (a repair costs a step): common prefix
        ok = 0
        for i in range(B):
            if prot[i]:
                n = min(len(res[a]["seqs"][i]), len(res[b]["seqs"][i]))
                ok += res[a]["seqs"][i][:n] == res[b]["seqs"][i][:n]
        return ok, int(prot.sum())

    dets = {"head": det("mg", "ao", head), "pipe": det_prefix("ao_pipe", "ao", head),
            "fused": det("mg_fused", "ao_fused", head),
            "other": det("mg_other", "ao_other", prot_all if other == "all" else prot_one) if "mg_other" in res
            else (0, 0)}
    times = {a: res[a]["ms"] for a in arms}
    times["e2e"] = e2e_ms
    red = sharding.reduce_run({a: res[a]["stats"] for a in arms}, keys, dets, {a: res[a]["tokens"] for a in arms},
                              times, probe=res["mg"]["seqs"][0] if ws > 1 else None, device="cuda")
    ao_probe = sharding.all_equal([sharding.digest(res["ao"]["seqs"][0])], device="cuda") if ws > 1 else None
    if rank != 0:
        if ws > 1:
            dist.destroy_process_group()
        return None
    stats = red["stats"]
    dh, do, dp, df = red["det"]["head"], red["det"]["other"], red["det"]["pipe"], red["det"]["fused"]
    ntok = red["tokens"]
    T = {a: red["times"][a] for a in arms}
    t_e2e = red["times"]["e2e"]
    tok = ws * B * K

    def summary(mg, ao, detv, prot_name):
        inc_mg = metrics.latency_increment(T[mg], T["bf16"])
        inc_ao = metrics.latency_increment(T[ao], T["bf16"])
        rt = metrics.rates(stats[mg])
        return {"protected": prot_name,
                "margingate_tok_s": round(tok / (T[mg] * 1e-3), 2),
                "always_on_tok_s": round(tok / (T[ao] * 1e-3), 2),
                "inc_margingate": round(inc_mg, 4), "inc_always_on": round(inc_ao, 4),
                "increment_ratio": (round(metrics.increment_ratio(inc_ao, inc_mg), 3)
                                    if stats[mg]["triggers"] > 0 and inc_mg > 0 else None),
                "trigger_pct": round(100 * rt["r_verify"], 3), "repair_pct": round(100 * rt["r_repair"], 4),
                "determinism_pct": round(100 * detv[0] / detv[1], 2) if detv[1] else None,
                "verifier_launches": stats[mg]["verifier_launches"], "catchup_tokens": stats[mg]["catchup_tokens"]}

    peaks = _peaks()
    hbm = peaks.get("hbm_gbs")
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if hbm else "fallback 6650 GB/s (B200_PROFILING.md)"
    hbm = hbm or 6650.0
    achieved = tim["gemm_bytes"] / (tim["gemm_ms"] * 1e-3) / 1e9 if tim["gemm_ms"] > 0 else None
    # the same launches less the measured floor of an event-bracketed launch
    # (an empty kernel of the GEMM's launch shape): what the raw per-launch
    # figure charges to launch processing rather than to the kernel
    floor_us = tim.get("floor_us")
    net_ms = tim["gemm_ms"] - (floor_us or 0.0) * 1e-3 * tim["gemm_launches"]
    achieved_net = tim["gemm_bytes"] / (net_ms * 1e-3) / 1e9 if floor_us and net_ms > 0 else None
    traffic = None
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "gemm_traffic.json"))).get("bytes_per_launch")
    except Exception:
        pass
    def pipe(a, prot_name, d):
        inc = (T[a] / ntok[a]) / (T["bf16"] / ntok["bf16"]) - 1
        return {"protected": prot_name, "always_on_tok_s": round(ntok[a] / (T[a] * 1e-3), 2),
                "inc_always_on": round(inc, 4), "repairs": stats[a]["repairs"],
                "determinism_pct": round(100 * d[0] / d[1], 2) if d and d[1] else None,
                "note": "MG_VERIFY_PIPELINED: the verifier of step t rides on step t+1's weight pass "
                        "(tokens = emitted - replaced); determinism = common prefix equal to the sync always-on run"}

    arms_out = {"bf16_tok_s": round(tok / (T["bf16"] * 1e-3), 2),
                "bf16_mid_decode_tok_s": round(tok / (T["bf16_mid"] * 1e-3), 2),
                "bf16_mid_decode_ctx": f"{ctx_mid + W}..{ctx_mid + W + K}", "tau": tau,
                "tau_source": "calibrated tau100 (seeds 10^6 + i)" if calib else "--tau",
                "headline": summary("mg", "ao", dh, args.protected)}
    if calib:
        arms_out["calibration"] = calib
    arms_out["headline"]["pipelined"] = pipe("ao_pipe", args.protected, dp)
    arms_out["headline"]["fused"] = {
        "margingate_tok_s": round(tok / (T["mg_fused"] * 1e-3), 2),
        "always_on_tok_s": round(tok / (T["ao_fused"] * 1e-3), 2),
        "inc_margingate": round(metrics.latency_increment(T["mg_fused"], T["bf16"]), 4),
        "inc_always_on": round(metrics.latency_increment(T["ao_fused"], T["bf16"]), 4),
        "trigger_pct": round(100 * metrics.rates(stats["mg_fused"])["r_verify"], 3),
        "determinism_pct": round(100 * df[0] / df[1], 2) if df[1] else None,
        "note": "MG_VERIFY_FUSED: every protected row's verifier token computed speculatively in the same "
                "weight pass; the gate selects which to commit (synchronous semantics)"}
    if full is not None:
        arms_out["full_decode"] = {"workload": full["workload"], "calibration": full["calibration"],
                                   **full["arms"]["one"], "protected": "one",
                                   "all_protected": full["arms"]["all"],
                                   "note": "rank 0; the whole decode, tau100 calibrated over the same length"}
    if w64 is not None:
        arms_out["llm42_window"] = {
            p: {"window": args.window, "steps": 2 * args.window, "tok_s": round(v[1] / (v[2] * 1e-3), 2),
                "inc": round((v[2] / v[1]) / (T["bf16"] / (B * K)) - 1, 4), **v[3],
                "note": "rank 0; inc per net committed token vs the BF16 arm per token"}
            for p, v in w64.items()}
    if "mg_other" in res:
        arms_out["other"] = summary("mg_other", "ao_other", do, other)
        if other == "all":   # determinism over every protected sequence of the batch (north star)
            arms_out["determinism_all_protected"] = {
                "margingate_pct": arms_out["other"]["determinism_pct"], "sequences": int(do[1]),
                "reference": "always-on run of the same batch (= the batch-1 reference, tests/test_gpu_engine.py)"}
        arms_out["other"]["pipelined"] = pipe("ao_pipe_other", other, None)
        arms_out["other"]["fused"] = {
            "always_on_tok_s": round(tok / (T["ao_fused_other"] * 1e-3), 2),
            "inc_always_on": round(metrics.latency_increment(T["ao_fused_other"], T["bf16"]), 4)}
    if ws > 1:
        arms_out["cross_rank_determinism"] = {
            "probe": "global request 0 decoded as row 0 (protected) on every rank, inside each rank's own batch",
            "identical_on_all_ranks": {"margingate": red["probe_identical"], "always_on": ao_probe}}
    arms_out["paper_context"] = ("A6000, bs=8, one protected request: 2.23x (8B) / 1.99x (14B) increment reduction "
                                 "at 18.56% / 15.05% triggers (PAPER.md:5, 285, 296) -- context, not the target")
    line = {
        "metric": METRIC,
        "value": round(tok / (T["mg"] * 1e-3), 2),
        "unit": "tok/s",
        "n_gpus": ws,
        "steps": K,
        "warmup": W,
        "ms_per_step": round(T["mg"] / K, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (random-init weights from the documented counter PRNG, uniform random prompts)",
        "config": {"workload": f"{args.model}-shaped {args.workload} decode, batch {B}/GPU, the last {K} decode "
                               f"steps (contexts {ctx0 + W}..{ctx0 + W + K}), protected={args.protected}, "
                               f"tau={'tau100' if calib else tau}",
                   "model": args.model, "global_batch": ws * B, "seq_len": ctx0 + W + K, "ctx_start": ctx0 + W,
                   "parallelism": f"request-sharded dp{ws}", "tau": tau, "protected": args.protected,
                   "l2": "inputs larger than L2 (15 GB of weights streamed per step)"},
        "arms": arms_out,
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1) if achieved else None, "peak": hbm,
                     "unit": "GB/s", "frac": round(achieved / hbm, 4) if achieved else None,
                     "traffic": traffic, "kernel": "k_gemm_tc (weight-streaming GEMM class, fast path)",
                     "peak_source": peak_src, "gemm_launches": tim["gemm_launches"],
                     "gemm_us_per_launch": round(1e3 * tim["gemm_ms"] / max(tim["gemm_launches"], 1), 2),
                     "launch_floor_us": round(floor_us, 2) if floor_us else None,
                     "net_of_launch_floor": ({"achieved": round(achieved_net, 1), "frac": round(achieved_net / hbm, 4),
                                              "note": "per-launch bytes / (event time - the event-bracketed launch "
                                                      "time of an empty kernel of the GEMM's shape, mgd_launch_floor)"}
                                             if achieved_net else None),
                     "gemm_ms_per_step": round(tim["gemm_ms"] / K, 4),
                     "attn_ms_per_step": round(tim["attn_ms"] / K, 4),
                     "fast_step_ms_timed_pass": round(tim["step_ms"] / max(tim["steps"], 1), 4),
                     # the whole pipelined BF16 step (CUDA graph, PDL) against the same peak:
                     # algorithmic bytes = weights once + every row's K/V context
                     "step": _step_roofline(shp, B, ctx0 + W + K // 2, T["bf16"] / K, hbm),
                     "step_mid_decode": _step_roofline(shp, B, ctx_mid + W + K // 2, T["bf16_mid"] / K, hbm),
                     # the synchronous verifier launches against the same peak --
                     # time = always-on step - BF16 step; bytes = weights once + the verified
                     # rows' shadow K/V (one protected row / all rows)
                     "verifier": {p: _verifier_roofline(shp, n, ctx0 + W + K // 2, (T[a] - T["bf16"]) / K, hbm)
                                  for p, n, a in (("one", 1, "ao" if args.protected == "one" else "ao_other"),
                                                  ("all", B, "ao_other" if args.protected == "one" else "ao"))
                                  if a in T}},
        "e2e": {"value": round(tok / (t_e2e * 1e-3), 2), "unit": "tok/s", "h2d_bytes_per_step": B * 5,
                "d2h_bytes_per_step": B * 5},
        "gpu_launches": res["mg"]["launches"],
        "clocks": res["mg"].get("clk"),
    }
    if paper is not None:
        r8 = paper["r"]
        tm = {n: r8[n][2] for n in r8}
        inc_mg = metrics.latency_increment(tm["margingate"], tm["bf16"])
        inc_ao = metrics.latency_increment(tm["always_on"], tm["bf16"])
        inc_tp = metrics.latency_increment(tm["margingate_tau_p"], tm["bf16"])
        pb = paper["batch"]
        line["arms"]["paper_protocol"] = {
            "batch": pb, "protected": "one", "tau": paper["tau100"], "tau_source": "calibrated tau100",
            "eps_pert_max": paper["calibration"]["eps_pert_max"], "tau_p": paper["calibration"]["tau_p"],
            "tok_s": {n: round(ws * r8[n][1]["tokens"] / (t * 1e-3), 2) for n, t in tm.items()},
            "inc_margingate": round(inc_mg, 4), "inc_always_on": round(inc_ao, 4),
            "increment_ratio": round(metrics.increment_ratio(inc_ao, inc_mg), 3) if inc_mg > 0.01 else None,
            "trigger_pct": round(100 * metrics.rates(r8["margingate"][1])["r_verify"], 3),
            "at_tau_p": {"inc_margingate": round(inc_tp, 4),
                         "increment_ratio": round(metrics.increment_ratio(inc_ao, inc_tp), 3) if inc_tp > 0.01 else None,
                         "trigger_pct": round(100 * metrics.rates(r8["margingate_tau_p"][1])["r_verify"], 3)},
            "protected_row_equals_reference": {n: r8[n][0][0] == r8["always_on"][0][0]
                                               for n in ("bf16", "margingate", "margingate_tau_p",
                                                         "margingate_token_only", "batch_invariant")},
            "token_only_repair": {"inc": round(metrics.latency_increment(tm["margingate_token_only"], tm["bf16"]), 4),
                                  "repairs": r8["margingate_token_only"][1]["repairs"],
                                  "note": "repair-action ablation, PAPER.md:317"},
            "batch_invariant": {"inc": round(metrics.latency_increment(tm["batch_invariant"], tm["bf16"]), 4),
                                "note": "global batch-invariant fast schedule at tau=0 (PAPER.md:227)"},
            "verify_modes": {n: {"inc": round((tm[n] / r8[n][1]["tokens"]) / (tm["bf16"] / (pb * K)) - 1, 4),
                              "trigger_pct": round(100 * metrics.rates(r8[n][1])["r_verify"], 3),
                              "repairs": r8[n][1]["repairs"],
                              "protected_row_equals_reference_prefix":
                                  r8[n][0][0][:min(len(r8[n][0][0]), len(r8["always_on"][0][0]))] ==
                                  r8["always_on"][0][0][:min(len(r8[n][0][0]), len(r8["always_on"][0][0]))]}
                          for n in ("margingate_pipelined", "always_on_pipelined", "margingate_fused",
                                    "always_on_fused")},
            "note": "rank 0's numbers (times not reduced over ranks)"}
        wseq, wtok, wms, wst = paper["window"]
        t_tok_bf16 = tm["bf16"] / (pb * K)
        inc_w = (wms / wtok) / t_tok_bf16 - 1
        n_ref = min(len(wseq[0]), len(r8["always_on"][0][0]))
        line["arms"]["paper_protocol"]["llm42_window"] = {
            "window": args.window, "steps": 2 * args.window, "tok_s": round(ws * wtok / (wms * 1e-3), 2),
            "inc": round(inc_w, 4),
            "increment_ratio_vs_margingate": round(inc_w / inc_mg, 3) if inc_mg > 0.01 else None,
            "net_tokens": wtok, **wst,
            "protected_row_equals_reference_prefix": wseq[0][:n_ref] == r8["always_on"][0][0][:n_ref],
            "note": "PAPER.md:251 LLM-42 K=64 analog: BF16 steps + windowed verify with rollback of the protected "
                    "row; inc per net committed token vs BF16 per token"}
    if ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, shp, tau)
    if ws > 1:
        dist.destroy_process_group()
    return line


def _step_roofline(shp, B, ctx, ms, peak_gbs):
    """SURVEY 8(d) per-step algorithmic bytes of the fast path: every weight
    streamed once (QKV, O, gate/up, down per layer + LM head) + each row's K/V
    over `ctx` keys; achieved = bytes / measured ms per step."""
    L, d, H, KV, hd, F, V = (shp[k] for k in ("n_layers", "d_model", "n_heads", "n_kv_heads", "head_dim", "d_ff",
                                                "vocab"))
    w = 2 * (L * ((H + 2 * KV) * hd * d + d * H * hd + 3 * F * d) + V * d)
    kv = B * ctx * L * 2 * KV * hd * 2
    gbs = (w + kv) / (ms * 1e-3) / 1e9
    return {"bytes": w + kv, "weights": w, "kv": kv, "ms": round(ms, 4), "achieved": round(gbs, 1),
            "frac": round(gbs / peak_gbs, 4)}


def _verifier_roofline(shp, rows, ctx, ms, peak_gbs):
    """Verifier launch of a step: weights once + `rows` rows'
    shadow K/V over `ctx` keys, in `ms` (always-on minus BF16 step time)."""
    r = _step_roofline(shp, rows, ctx, ms, peak_gbs)
    r["rows"] = rows
    return r


def _oracle_sample(shp, prompt_len, steps, tau, budget_s, rows=1, sched_batch=1, model=None):
    """The oracle (as it stands) decoding `rows` rows: prefill `prompt_len`
    tokens (untimed), then up to `steps` MarginGate decode steps with the
    oracle's batch-shaped plan of batch `sched_batch`, timed; returns (tokens,
    seconds).  The oracle decodes rows independently, so a bounded sample of
    rows of a large batch costs what those rows cost inside it."""
    import oracle
    m = model or oracle.Model(shp)
    st = oracle.State(m, rows, prompt_len + steps + 2)
    det = oracle.det_sched()
    for r in range(rows):
        st.prefill(r, [int(t) for t in np.random.default_rng(7 + r).integers(0, shp["vocab"], prompt_len)], det)
    t0 = time.time()
    n = 0
    for _ in range(steps):
        st.step(list(range(rows)), [1] * rows, tau, oracle.fast_sched(sched_batch), det)
        n += rows
        if time.time() - t0 > budget_s:
            break
    dt = time.time() - t0
    st.close()
    if model is None:
        m.close()
    return n, dt


def _oracle_tiny(bs, tau=0.3):
    """BASELINE configs[0] in full: the tiny decoder, 8 prompts x 32 greedy
    tokens, at batch 1 (each prompt alone) or batch 8; tokens/s of the timed
    decode steps (prefill untimed)."""
    import oracle

    from paper_2605_30218_b200 import inputs
    shp = inputs.shape("tiny")
    m = oracle.Model(shp)
    det = oracle.det_sched()
    prompts = inputs.prompts(8, inputs.ragged_lengths(8, 8, 23), shp["vocab"])
    n, dt = 0, 0.0
    for g in range(0, 8, bs):
        grp = prompts[g:g + bs]
        st = oracle.State(m, len(grp), 64)
        for i, p in enumerate(grp):
            st.prefill(i, p, det)
        t0 = time.time()
        for _ in range(31):
            st.step(list(range(len(grp))), [1] * len(grp), tau, oracle.fast_sched(len(grp)), det)
        dt += time.time() - t0
        n += 31 * len(grp)
        st.close()
    m.close()
    return n, dt


def cpu_baseline(args, shp, tau):
    cores = len(os.sched_getaffinity(0))
    os.environ["OMP_NUM_THREADS"] = str(cores)
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 0
    need = 2.2 * 2 * (shp["vocab"] * shp["d_model"] * 2 + shp["n_layers"] * (
        (shp["n_heads"] + 2 * shp["n_kv_heads"]) * shp["head_dim"] * shp["d_model"] +
        shp["d_model"] * shp["n_heads"] * shp["head_dim"] + 3 * shp["d_ff"] * shp["d_model"]))
    if avail and avail < need:
        return {"value": None, "unit": "tok/s", "cores": cores, "kind": "oracle",
                "sample": f"skipped: {avail / 2**30:.0f} GiB host RAM < {need / 2**30:.0f} GiB needed"}
    n, dt = _oracle_sample(shp, 8, 8, tau, 20.0)   # ~10-30 s of CPU work
    out = {"value": round(n / dt, 5), "unit": "tok/s", "cores": cores, "kind": "oracle",
           "sample": f"{args.model}-shaped, 1 row, {n} MarginGate decode steps (tau={tau}) after an 8-token "
                     f"deterministic prefill; {dt:.1f} s of CPU time"}
    # SURVEY 8(d) samples: the same model inside a batch of 64 (two rows of one
    # step, the oracle's batch-64 reduction plan) and BASELINE configs[0] in full
    n64, dt64 = _oracle_sample(shp, 8, 1, tau, 20.0, rows=2, sched_batch=64)
    out["samples"] = {
        f"{args.model}_bs64": {"value": round(n64 / dt64, 5), "unit": "tok/s",
                               "sample": f"2 of the 64 rows of one step (batch-64 plan), {dt64:.1f} s"}}
    for bs in (1, 8):
        nt, dtt = _oracle_tiny(bs)
        out["samples"][f"tiny_bs{bs}"] = {"value": round(nt / dtt, 2), "unit": "tok/s",
                                          "sample": f"configs[0]: 8 prompts x 32 greedy tokens at batch {bs}, "
                                                    f"tau 0.3, {dtt:.2f} s"}
    return out


def _launch_floor(eng, reps=50):
    """Mean CUDA-event-bracketed time of an empty kernel with the fast-path
    GEMM's launch shape (148 x 192 threads, the 64-token tile's 197744 B of
    shared memory) on the engine's stream (include/mg_debug.h)."""
    import ctypes as C

    from paper_2605_30218_b200._lib import lib
    us = C.c_float(0.0)
    if lib().mgd_launch_floor(197744, reps, C.c_void_p(eng.stream.cuda_stream), C.byref(us)) != 0:
        return None
    return float(us.value)


def run_reference(args):
    """The oracle as it stands on the host cores, on the GPU arm's workload:
    the protected request (row 0) decoded with the oracle's batch-shaped plan
    of the bench batch.  Its threshold is the oracle's own perturbation bound
    (the rule the GPU arm's calibration follows): the largest
    |logit(batch plan) - logit(pinned plan)| over the warm-up steps, measured
    by a second oracle state teacher-forced on the same tokens; the verifier
    runs on the steps whose margin is below it.  Bounded sample: one row of the
    batch (the oracle decodes rows independently) after an 8-token prefill --
    a prefill of the GPU arm's context (615 tokens) would take ~40 min of 8B
    oracle forwards; the decode step's oracle cost is dominated by the weight
    GEMVs (15 GMAC per token), attention over 640 keys adds ~1%."""
    ws, rank, _ = _dist()
    if rank != 0:
        return None
    from paper_2605_30218_b200 import inputs
    shp = inputs.shape(args.model)
    cores = len(os.sched_getaffinity(0))
    os.environ["OMP_NUM_THREADS"] = str(cores)
    import oracle
    m = oracle.Model(shp)
    p = [int(t) for t in np.random.default_rng(7).integers(0, shp["vocab"], 8)]
    st = oracle.State(m, 1, 8 + args.steps + args.warmup + 2)
    det = oracle.det_sched()
    st.prefill(0, p, det)
    fast = oracle.fast_sched(args.batch)
    pin = oracle.State(m, 1, 8 + args.warmup + 2)   # the pinned plan on the same tokens (warm-up only)
    pin.prefill(0, p, det)
    eps = 0.0
    for _ in range(args.warmup):
        ra = st.step([0], [1], 0.0, fast, det, want_logits=True)
        rd = pin.step([0], [1], 0.0, det, det, forced_out=[int(ra["out"][0])], want_logits=True)
        eps = max(eps, float(np.abs(ra["logits"][0] - rd["logits"][0]).max()))
    pin.close()
    tau = args.tau if args.tau is not None else eps
    t0 = time.time()
    trig = 0
    for _ in range(args.steps):
        trig += st.step([0], [1], tau, fast, det)["n_trig"]
    dt = time.time() - t0
    v = args.steps / dt
    sample = (f"the protected request (row 0 of the {args.batch}-row batch, the oracle's batch-{args.batch} "
              f"reduction plan), {args.steps} timed MarginGate steps at tau={tau:.4g} ({trig} verifier runs) "
              f"after an 8-token prefill; the GPU arm's context 615..640 is not prefilled here (~40 min of "
              f"oracle forwards; the step cost is dominated by the 15 GMAC of weight GEMVs, attention adds ~1%)")
    return {"impl": "reference", "metric": METRIC, "value": round(v, 5), "unit": "tok/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * dt / args.steps, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": f"{args.model}-shaped {args.workload} decode, batch {args.batch}/GPU, "
                                   f"protected=one, tau={tau:.4g} (the oracle's eps_pert over the warm-up)",
                       "model": args.model, "global_batch": args.batch, "parallelism": "dp1 (rank 0 only)",
                       "tau": tau, "protected": "one", "sample": sample},
            "cpu_baseline": {"value": round(v, 5), "unit": "tok/s", "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": round(v, 5), "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def _decode_run(eng, prompts, tau, prot, W, K, eps=None, timed=False, flips=None, pipelined=False, fused=False):
    """Fresh prefill of `prompts`, W + K decode steps at threshold tau; eps (a
    list) collects eps_pert per (row, step) -- only valid at tau = inf with
    every row protected, where the verifier's rank k is row k.  flips (a
    list) collects (fast margin g, fast token != verifier token) per (row,
    step) of the gated rows -- at tau = inf every step is synchronous (the
    committed prefix is the reference's)."""
    import torch
    B = len(prompts)
    V = eng.shape["vocab"]
    out = torch.empty(B, dtype=torch.int32, device="cuda")
    kind = torch.empty(B, dtype=torch.uint8, device="cuda")
    rows = list(range(B))
    for i in range(B):
        try:
            eng.release(i)
        except Exception:
            pass
    eng.set_policy(verify_mode=1 if pipelined else (2 if fused else 0))
    seqs = [[eng.prefill(i, p)] for i, p in enumerate(prompts)]
    s0 = eng.stats()
    capf = capv = None
    replaced = 0
    if eps is not None:
        capf = torch.empty((B, V), dtype=torch.float32, device="cuda")
        capv = torch.empty((B, V), dtype=torch.float32, device="cuda")
        eng.capture_logits(capf)
        eng.capture_verifier_logits(capv)
    ms = 0.0
    for k in range(W + K):
        if timed and k == W:
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(eng.stream)
        eng.step(rows, prot, tau, out, kind)
        o = out.cpu().numpy()
        kk = kind.cpu().numpy() if pipelined else None
        for b in range(B):
            if pipelined and kk[b] == 4:   # MG_VERIFY_PIPELINED: replaces the last (tentative) token
                seqs[b][-1] = int(o[b])
                replaced += k >= W
            else:
                seqs[b].append(int(o[b]))
        if flips is not None:
            r = eng.last_step(B)
            flips.extend((float(r["g"][b]), bool(r["f_tok"][b] != r["v_tok"][b])) for b in range(B) if r["trig"][b])
        if eps is not None:
            idx = torch.topk(capv, 50, dim=1).indices          # reference top-50
            d = (capf.gather(1, idx) - capv.gather(1, idx)).abs().amax(dim=1)
            eps.extend(d.cpu().tolist())
    if timed:
        e1.record(eng.stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    if eps is not None:
        eng.capture_logits(None)
        eng.capture_verifier_logits(None)
    if pipelined:
        pos, last, _ = eng.verify_window(rows)
        for b in range(B):
            n = int(pos[b]) - len(prompts[b]) + 1
            del seqs[b][n:]
            seqs[b][-1] = int(last[b])
        eng.set_policy(verify_mode=0)
    if fused:
        eng.set_policy(verify_mode=0)
    s1 = eng.stats()
    st = {k: s1[k] - s0[k] for k in ("protected_rows", "triggers", "repairs")}
    st["tokens"] = B * K - replaced
    return seqs, st, ms


def _window_run(eng, prompts, prot, W, K, window):
    """LLM-42-style comparator:
    pure BF16 steps, and every `window` steps mg_verify_window on the
    protected rows (rollback at the first disagreement).  Fresh prefill, W
    warm-up steps (verified at their end), then K timed steps ending with a
    verify.  Returns (verified sequences of the rows, net committed tokens in
    the timed region, ms, window stats)."""
    import torch
    B = len(prompts)
    P = [len(p) for p in prompts]
    rows = list(range(B))
    vrows = [i for i in rows if prot[i]]
    for i in range(B):
        try:
            eng.release(i)
        except Exception:
            pass
    seqs = [[eng.prefill(i, p)] for i, p in enumerate(prompts)]
    hist = []

    def flush():
        o = torch.stack(hist).cpu().numpy() if hist else np.empty((0, B), np.int32)
        hist.clear()
        for b in range(B):
            seqs[b].extend(int(t) for t in o[:, b])
        pos, last, rb = eng.verify_window(vrows)
        for j, b in enumerate(vrows):
            n = int(pos[j]) - P[b] + 1
            del seqs[b][n:]
            seqs[b][-1] = int(last[j])

    out_bufs = [torch.empty(B, dtype=torch.int32, device="cuda") for _ in range(W + K)]
    it = iter(out_bufs)

    def step_into():
        o = next(it)
        eng.step(rows, None, 0.0, o)
        return o

    # warm-up: W steps then a verify
    for _ in range(W):
        hist.append(step_into())
    flush()
    n0 = sum(len(s) for s in seqs)
    s0 = eng.stats()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(eng.stream)
    for k in range(K):
        hist.append(step_into())
        if (k + 1) % window == 0 or k == K - 1:
            flush()
    e1.record(eng.stream)
    torch.cuda.synchronize()
    s1 = eng.stats()
    st = {k: s1[k] - s0[k] for k in ("window_rows", "rollbacks", "rolled_back_tokens", "catchup_tokens")}
    return seqs, sum(len(s) for s in seqs) - n0, e0.elapsed_time(e1), st


def calibrate(eng, prompts, W, K):
    """SURVEY A22 / PAPER.md:260-265, 402: eps_pert on calibration prompts
    (tau = inf, all rows protected: batched fast vs deterministic verifier
    logits on the same committed prefix, reference top-50), tau_p = 2 max eps,
    grid {0, tau_p 2^k (k = -3..3)}; tau100 = smallest grid point whose
    protected sequences all equal the tau = inf run (metrics.tau100)."""
    from paper_2605_30218_b200 import inputs, metrics
    B = len(prompts)
    prot = inputs.protected_mask(B, "all")
    eps, fl = [], []
    ref, _, _ = _decode_run(eng, prompts, math.inf, prot, W, K, eps=eps, flips=fl)
    tau_p = metrics.pert_tau(eps)
    grid = sorted(set([0.0] + [tau_p * 2.0 ** k for k in range(-3, 4)]))
    ev = [g for g, f in fl if f]
    rows = []
    for tau in grid:
        seqs, st, _ = _decode_run(eng, prompts, tau, prot, W, K)
        rows.append({"tau": tau, "det_pct": round(100 * metrics.seq_determinism(seqs, ref), 2),
                     "trigger_pct": round(100 * metrics.rates(st)["r_verify"], 3)})
    t100 = metrics.tau100([(r["tau"], r["det_pct"] / 100) for r in rows])
    return {"eps_pert_max": max(eps), "eps_pert_p50": float(np.median(eps)), "samples": len(eps),
            "tau_p": tau_p, "grid": rows, "tau100": t100,
            # synchronous flip rate and trigger recall (tab:hetero)
            "sync_flip_rate": len(ev) / len(fl) if fl else None, "flip_events": len(ev),
            "recall": {f"{t:.4g}": metrics.margin_recall(ev, t) for t in grid if t > 0} if ev else None}


def kv_trace(eng, shp, B, P, steps, trials):
    """Row 0 decoded at tau = 0 inside a batch of B (fast cache) vs alone at
    tau = inf (the reference; its shadow cache is the deterministic K/V of the
    reference tokens): E^K_p, E^V_p per layer (metrics.kv_deviation) over the
    decoded positions, split by Delta = p - p_div."""
    import torch

    from paper_2605_30218_b200 import inputs, metrics
    L = shp["n_layers"]
    out = torch.empty(B, dtype=torch.int32, device="cuda")
    layers = sorted({0, L // 2, L - 1})
    pre, at, post, n_div = [], [], [], 0
    for tr in range(trials):
        prompts = inputs.prompts(B, P, shp["vocab"], seed=4000 + 97 * tr)
        for i in range(B):
            try:
                eng.release(i)
            except Exception:
                pass
        seq = [eng.prefill(i, p) for i, p in enumerate(prompts)][:1]
        for _ in range(steps):
            eng.step(list(range(B)), None, 0.0, out)
            seq.append(int(out[0].item()))
        fast = [eng.read_column(0, 0, P + i) for i in range(steps)]
        for i in range(B):
            eng.release(i)
        ref = [eng.prefill(0, prompts[0])]
        o1 = out[:1]
        for _ in range(steps):
            eng.step([0], [1], math.inf, o1)
            ref.append(int(o1[0].item()))
        shadow = [eng.read_column(1, 0, P + i) for i in range(steps)]
        eng.release(0)
        d = metrics.first_divergence(seq, ref)
        ek, ev = metrics.kv_deviation(fast, shadow)
        p_div = None if d is None else P + d       # the first column whose input token differs (token d sits at P + d)
        if p_div is not None:
            n_div += 1
        for i in range(steps):
            row = (ek[i][layers].tolist(), ev[i][layers].tolist())
            if p_div is None or P + i < p_div:
                pre.append(row)
            elif P + i == p_div:
                at.append(row)
            else:
                post.append(row)

    def agg(rows):
        if not rows:
            return None
        a = np.array(rows)  # [n][2][layers]
        return {"K_max": [round(float(x), 5) for x in a[:, 0].max(0)],
                "V_max": [round(float(x), 5) for x in a[:, 1].max(0)],
                "K_median": [round(float(x), 5) for x in np.median(a[:, 0], 0)],
                "V_median": [round(float(x), 5) for x in np.median(a[:, 1], 0)], "n": len(rows)}
    return {"layers": layers, "trials": trials, "batch": B, "divergent_trials": n_div,
            "before_divergence": agg(pre), "at_divergence": agg(at), "after_divergence": agg(post),
            "paper_context": "fig:err_vs_dist / tab:kv_struct (PAPER.md:71-80, 474): deviations stay at the "
                             "pre-divergence noise floor and spike at Delta = 0 -- Llama-8B on A6000"}


def run_sweep(args):
    """calibrate tau on calibration seeds (1000 + i),
    then evaluate tau in {0, tau100, inf} on the disjoint bench seeds (7 + i)
    with one protected row and with all rows protected."""
    from paper_2605_30218_b200 import inputs, metrics
    from paper_2605_30218_b200.engine import Engine

    shp = inputs.shape(args.model)
    B, K, W = args.batch, args.steps, args.warmup
    prompt_len, _ = inputs.WORKLOADS[args.workload]
    eng = Engine(shp, max_batch=B, max_slots=B, max_seq=prompt_len + W + K + 4, page_size=64)
    cal = calibrate(eng, inputs.prompts(B, prompt_len, shp["vocab"], seed=CALIB_SEED), W, K)
    t_eval = cal["tau100"] if cal["tau100"] is not None else math.inf
    ev = inputs.prompts(B, prompt_len, shp["vocab"], seed=7)
    evals = {}
    for pname in ("one", "all"):
        prot = inputs.protected_mask(B, pname)
        res = {name: _decode_run(eng, ev, tau, prot, W, K, timed=True)
               for name, tau in (("bf16", 0.0), ("margingate", t_eval), ("always_on", math.inf))}
        ref_e = res["always_on"][0]
        pr = [i for i in range(B) if prot[i]]
        tm = {n: r[2] for n, r in res.items()}
        evals[pname] = {
            "tau": t_eval,
            "tok_s": {n: round(B * K / (t * 1e-3), 2) for n, t in tm.items()},
            "inc_margingate": round(metrics.latency_increment(tm["margingate"], tm["bf16"]), 4),
            "inc_always_on": round(metrics.latency_increment(tm["always_on"], tm["bf16"]), 4),
            "trigger_pct": round(100 * metrics.rates(res["margingate"][1])["r_verify"], 3),
            "determinism_pct": {n: round(100 * metrics.seq_determinism([res[n][0][i] for i in pr],
                                                                       [ref_e[i] for i in pr]), 2)
                                for n in ("bf16", "margingate")},
        }
    # SURVEY A24 (seq. det. over >= 120 protected sequences):
    # every row protected, `trials` disjoint evaluation batches (seeds 7 + B j)
    trials = {"tau": t_eval, "tau_p": cal["tau_p"], "batches": args.trials, "protected_sequences": 0,
              "deterministic": {"bf16": 0, "margingate": 0, "margingate_tau_p": 0}, "triggers": 0,
              "triggers_tau_p": 0, "protected_steps": 0}
    pall = inputs.protected_mask(B, "all")
    for j in range(args.trials):
        evj = inputs.prompts(B, prompt_len, shp["vocab"], seed=7 + B * j)
        ref_j = _decode_run(eng, evj, math.inf, pall, W, K)[0]
        for n, tau in (("bf16", 0.0), ("margingate", t_eval), ("margingate_tau_p", cal["tau_p"])):
            sj, stj, _ = _decode_run(eng, evj, tau, pall, W, K)
            trials["deterministic"][n] += sum(1 for i in range(B) if sj[i] == ref_j[i])
            if n == "margingate":
                trials["triggers"] += stj["triggers"]
                trials["protected_steps"] += stj["protected_rows"]
            if n == "margingate_tau_p":
                trials["triggers_tau_p"] += stj["triggers"]
        trials["protected_sequences"] += B
    trials["determinism_pct"] = {n: round(100 * v / max(trials["protected_sequences"], 1), 2)
                                 for n, v in trials["deterministic"].items()}
    trials["trigger_pct"] = round(100 * trials["triggers"] / max(trials["protected_steps"], 1), 3)
    trials["trigger_pct_tau_p"] = round(100 * trials["triggers_tau_p"] / max(trials["protected_steps"], 1), 3)
    evals["trials_all_protected"] = trials
    eng.close()
    # NEXT-3 (App. C tab:hetero): trigger check on same-prompt-replicated
    # (homogeneous) vs mixed prompts of ragged lengths (heterogeneous; per-row
    # positions, the paged cache needs no padding)
    het = {}
    eng = Engine(shp, max_batch=B, max_slots=B, max_seq=prompt_len * 3 // 2 + W + K + 4, page_size=64)
    homo_p = inputs.prompts(1, prompt_len, shp["vocab"], seed=2000) * B
    lens = inputs.ragged_lengths(B, prompt_len // 2, prompt_len * 3 // 2, seed=2001)
    het_p = inputs.prompts(B, lens, shp["vocab"], seed=3000)
    for name, ps in (("homogeneous", homo_p), ("heterogeneous", het_p)):
        fl = []
        _decode_run(eng, ps, math.inf, inputs.protected_mask(B, "all"), W, K, flips=fl)
        ev = [g for g, f in fl if f]
        het[name] = {"sync_flip_rate": round(len(ev) / len(fl), 5), "flip_events": len(ev), "samples": len(fl),
                     "recall": {f"{t:.4g}": metrics.margin_recall(ev, t)
                                for t in (cal["tau_p"] / 2, cal["tau_p"], 2 * cal["tau_p"]) if t > 0} if ev else None}
    het["lengths"] = lens
    eng.close()
    # NEXT-4 second half (fig:err_vs_dist, tab:kv_struct): K/V deviation of the
    # protected request's batched BF16 trajectory from the deterministic reference,
    # per layer and position, aligned to the first token divergence
    eng = Engine(shp, max_batch=B, max_slots=B, max_seq=prompt_len + W + K + 4, page_size=64)
    kvd = kv_trace(eng, shp, B, prompt_len, W + K, trials=4)
    eng.close()
    return {"metric": "tau calibration sweep (SURVEY 8(f) NEXT-1, A22)", "model": args.model,
            "hetero_check": het, "kv_deviation": kvd,
            "workload": f"{args.workload}-shaped prompt {prompt_len}, {K} timed decode steps after {W}, batch {B}",
            "calibration": {"seeds": "10^6 + i", **cal},
            "evaluation": {"seeds": "7 + i", **evals},
            "paper_context": "tab:pareto / tab:eps_pert (PAPER.md:260-265, 402-421): tau100 from a doubling "
                             "sweep on calibration prompts, A6000 -- context, not the target"}


def run_full_decode(args, pnames=("one", "all"), eng=None):
    """The whole MATH500-shaped decode at the headline batch (prompt 128, all
    512 decode steps, SURVEY 8(d) "tok/s = emitted decode tokens / decode time"):
    contexts 128..640 cross the verifier's 512-key split, so the fast path's
    batch-shaped attention differs from the verifier in the second half.  tau100
    calibrated over the same decode length on seeds 10^6 + i; arms BF16,
    MarginGate and always-on, synchronous and fused, one and all rows protected."""
    from paper_2605_30218_b200 import inputs, metrics
    from paper_2605_30218_b200.engine import Engine

    shp = inputs.shape(args.model)
    B, W = args.batch, 3
    prompt_len, decode_len = inputs.WORKLOADS[args.workload]
    K = decode_len - W
    own = eng is None
    if own:
        eng = Engine(shp, max_batch=B, max_slots=B, max_seq=prompt_len + decode_len + 2, page_size=64)
    cal = calibrate(eng, inputs.prompts(B, prompt_len, shp["vocab"], seed=CALIB_SEED), W, K)
    t100 = cal["tau100"] if cal["tau100"] is not None else math.inf
    ev = inputs.prompts(B, prompt_len, shp["vocab"], seed=7)
    out = {}
    for pname in pnames:
        prot = inputs.protected_mask(B, pname)
        r = {n: _decode_run(eng, ev, t, prot, W, K, timed=True, fused=f)
             for n, t, f in (("bf16", 0.0, False), ("margingate", t100, False), ("always_on", math.inf, False),
                             ("margingate_fused", t100, True), ("always_on_fused", math.inf, True),
                             # the argmax-bound threshold 2 max eps: covers every flip
                             # the calibration saw, at a higher trigger rate than tau100
                             ("margingate_tau_p", cal["tau_p"], False))}
        pr = [i for i in range(B) if prot[i]]
        ref = r["always_on"][0]
        out[pname] = {
            "tok_s": {n: round(B * K / (v[2] * 1e-3), 2) for n, v in r.items()},
            "inc": {n: round(metrics.latency_increment(v[2], r["bf16"][2]), 4) for n, v in r.items() if n != "bf16"},
            "trigger_pct": round(100 * metrics.rates(r["margingate"][1])["r_verify"], 3),
            "trigger_pct_tau_p": round(100 * metrics.rates(r["margingate_tau_p"][1])["r_verify"], 3),
            "determinism_pct": {n: round(100 * metrics.seq_determinism([r[n][0][i] for i in pr],
                                                                       [ref[i] for i in pr]), 2)
                                for n in ("bf16", "margingate", "margingate_fused", "margingate_tau_p")}}
        inc_mg, inc_ao = out[pname]["inc"]["margingate"], out[pname]["inc"]["always_on"]
        out[pname]["increment_ratio"] = round(metrics.increment_ratio(inc_ao, inc_mg), 3) if inc_mg > 0.01 else None
    if own:
        eng.close()
    return {"metric": "full-decode tok/s, increments, triggers, determinism", "model": args.model,
            "workload": f"{args.workload}-shaped prompt {prompt_len}, {K} timed decode steps after {W} "
                        f"(contexts {prompt_len + W}..{prompt_len + decode_len}), batch {B}",
            "calibration": {k: cal[k] for k in ("eps_pert_max", "tau_p", "tau100", "sync_flip_rate", "flip_events")},
            "arms": out}


def run_batch_scaling(args):
    """tab:batch_scaling analog: latency increment over BF16
    of MarginGate (tau100 calibrated per batch on seeds 10^6 + i) and of
    always-on verification, synchronous and fused verify modes, one protected
    request, at batch 8 / 16 / 32 / 64."""
    from paper_2605_30218_b200 import inputs, metrics
    from paper_2605_30218_b200.engine import Engine

    shp = inputs.shape(args.model)
    K, W = args.steps, args.warmup
    prompt_len, decode_len = inputs.WORKLOADS[args.workload]
    ctx0 = prompt_len + decode_len // 2 - W
    rows = []
    for B in (8, 16, 32, 64):
        eng = Engine(shp, max_batch=B, max_slots=B, max_seq=ctx0 + W + K + 2, page_size=64)
        cal = calibrate(eng, inputs.prompts(B, ctx0, shp["vocab"], seed=CALIB_SEED), 3, min(K, 16))
        t100 = cal["tau100"] if cal["tau100"] is not None else math.inf
        ev = inputs.prompts(B, ctx0, shp["vocab"], seed=7)
        p1 = inputs.protected_mask(B, "one")
        r = {n: _decode_run(eng, ev, t, p1, W, K, timed=True, fused=f)
             for n, t, f in (("bf16", 0.0, False), ("margingate", t100, False), ("always_on", math.inf, False),
                             ("margingate_fused", t100, True), ("always_on_fused", math.inf, True))}
        eng.close()
        inc = {n: round(metrics.latency_increment(r[n][2], r["bf16"][2]), 4) for n in r if n != "bf16"}
        rows.append({"batch": B, "tau100": t100, "eps_pert_max": cal["eps_pert_max"],
                     "bf16_tok_s": round(B * K / (r["bf16"][2] * 1e-3), 2), "inc": inc,
                     "trigger_pct": round(100 * metrics.rates(r["margingate"][1])["r_verify"], 3),
                     "protected_row_equals_reference": {n: r[n][0][0] == r["always_on"][0][0]
                                                        for n in ("bf16", "margingate", "margingate_fused")}})
    return {"metric": "batch-scaling latency increments (tab:batch_scaling analog)", "model": args.model,
            "workload": f"{args.workload}-shaped, context {ctx0 + W}..{ctx0 + W + K}, one protected request",
            "rows": rows,
            "paper_context": "PAPER.md:331-334 (A6000, 8B): LLM-42 64.6/69.0/73.8/106.5% vs MarginGate "
                             "29.0/45.4/61.6/73.6% at bs 8/16/32/64 -- context, not the target"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=32)
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="llama8b")
    ap.add_argument("--workload", default="math500")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--tau", type=float, default=None, help="fixed threshold (default: calibrated tau100)")
    ap.add_argument("--protected", default="one", choices=["one", "all"])
    ap.add_argument("--quick", action="store_true", help="skip the other protection mode")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--paper-batch", type=int, default=8, help="batch of the paper-protocol arm (0: off)")
    ap.add_argument("--window", type=int, default=64, help="LLM-42 verify window (PAPER.md:251 K=64)")
    ap.add_argument("--sweep", action="store_true", help="tau calibration sweep report (NEXT-1) instead of the "
                                                          "bench line")
    ap.add_argument("--trials", type=int, default=15, help="--sweep: evaluation batches (B x trials protected "
                                                          "sequences, SURVEY A24)")
    ap.add_argument("--no-full-decode-arm", dest="full_decode_arm", action="store_false",
                    help="skip the whole-decode arm of the bench line")
    ap.add_argument("--full-decode", action="store_true", help="whole-decode report (all decode steps) instead "
                                                                 "of the bench line")
    ap.add_argument("--batch-scaling", action="store_true", help="tab:batch_scaling analog report instead of the "
                                                                   "bench line")
    args = ap.parse_args()
    assert args.warmup >= 3, "W >= 3"
    if args.full_decode:
        line = run_full_decode(args)
    elif args.batch_scaling:
        line = run_batch_scaling(args)
    elif args.sweep:
        line = run_sweep(args)
    else:
        line = run_reference(args) if args.impl == "reference" else run_gpu(args)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
