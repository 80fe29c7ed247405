#!/usr/bin/env python
"""Benchmark: deterministic decode tok/s at Llama-3-8B shape, plus the receipt replay rate.

Workload (BASELINE.json configs[1]): Llama-3-8B-shape random-init bf16 model, greedy decode, batch 1
per GPU, prompt 512 / gen 256. One bench "step" = one generate() of that batch (prefill of the
prompt + 256 sampled tokens with their f32 logits trace). N GPUs = N independent replicas (weak
scaling, no collective on the data path). See DESIGN.md §6 for the measurement definitions.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--batch B --prompt P --gen T]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "deterministic decode tok/s at Llama-3-8B shape; bit-exact receipt replay rate"
HBM_FALLBACK = 6650.0   # GB/s, B200_PROFILING.md fallback when MEASURED_PEAKS.json is absent
CLASS_NAMES = ["norm", "qkv_gemm", "attention", "o_gemm", "gate_up_gemm", "down_gemm", "lm_head_gemm", "sample"]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="llama3-8b:bench")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--prompt", type=int, default=512)
    ap.add_argument("--gen", type=int, default=256)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-baseline", default="auto", choices=["auto", "off"])
    ap.add_argument("--sweep", default="auto", choices=["auto", "off"],
                    help="N=1: decode-step tok/s and step roofline at batch 1/8/64/256 (context 640)")
    ap.add_argument("--traffic", default="auto", choices=["auto", "off"],
                    help="N=1: DRAM bytes of one gate/up launch, measured by ncu in a subprocess")
    ap.add_argument("--cpu-sample-prompt", type=int, default=4)
    ap.add_argument("--cpu-sample-gen", type=int, default=2)
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return HBM_FALLBACK, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.proc, self.lines = device, None, []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None, "reasons": sorted(reasons),
                "samples": len(sm)}


def step_bytes(info, batch: int, prompt: int, gen: int) -> float:
    """Algorithmic HBM bytes of one decode step: every bf16 weight once, plus per
    request the KV read (mean context), KV write, embedding row and f32 logits write."""
    d, L, hq, hkv, hd, F, V = (info.d_model, info.n_layers, info.n_heads, info.n_kv_heads, info.head_dim, info.ffn,
                               info.vocab)
    weights = 2.0 * (L * (d * (hq + 2 * hkv) * hd + hq * hd * d + 3 * d * F + 2 * d) + d + 2 * V * d) - 2.0 * V * d
    kv_per_pos = L * 2 * hkv * hd * 2
    mean_ctx = prompt + gen / 2.0
    per_req = kv_per_pos * mean_ctx + kv_per_pos + 2 * d + 4 * V
    return weights + batch * per_req


def batch_sweep(model: str, eng_b1, batches=(1, 8, 64, 256), ctx: int = 640):
    """Decode-step throughput vs batch (config 3's batch sizes) on a second engine with 256 slots:
    CUDA-graph step time with every column at context `ctx` (detgpu_profile_graph), tok/s and the
    step's HBM roofline fraction (SURVEY.md §8(d) bytes). Receipt identity across these batch sizes
    is tests/test_gpu_determinism.py's job; this is throughput only."""
    import ctypes as C

    from paper_2602_00182_b200 import _lib as L
    from paper_2602_00182_b200.detcore import Engine

    info = eng_b1.info
    peak, _ = peaks()
    eng = Engine(model, "b200", max_batch=max(batches), max_context=max(ctx + 1, 768))
    out = {"ctx": ctx, "what": "CUDA-graph decode step, every column at context ctx; step_frac = SURVEY §8(d) bytes "
                              "/ step time / measured HBM peak"}
    try:
        for b in batches:
            ms = C.c_float()
            L.check(L.lib.detgpu_profile_graph(eng.h, b, ctx, 0, 10, C.byref(ms)), eng.h)
            sb = step_bytes(info, b, ctx, 0)
            out[str(b)] = {"ms_per_step": round(ms.value, 4), "tok_s": round(b / ms.value * 1e3, 1),
                           "step_frac": round(sb / (ms.value / 1e3) / 1e9 / peak, 4)}
    finally:
        eng.close()
    return out


def cpu_oracle_sample(model: str, prompt_len: int, gen: int, vocab_hint: int = 128256):
    """Time the CPU oracle (a C++ restatement of the path; the reference itself has no transformer)
    on a bounded sample of the workload: one request, prompt_len prompt tokens, gen decoded."""
    from oracle import oracle as O

    threads = os.cpu_count() or 1
    O.lib().orc_set_threads(threads)
    t0 = time.perf_counter()
    m = O.Llama(model)
    t_init = time.perf_counter() - t0
    prompt = np.random.default_rng(7).integers(0, m.V, prompt_len).astype(np.uint32)
    t1 = time.perf_counter()
    m.generate(prompt, max_tokens=gen)
    dt = time.perf_counter() - t1
    del m
    return {"value": gen / dt, "unit": "tok/s", "cores": threads, "kind": "port",
            "sample": f"{model}: 1 request, prompt {prompt_len} tokens (one multi-column prefill) + {gen} generated "
                      f"tokens, {dt:.1f} s; weight generation {t_init:.1f} s excluded. NOT the GPU arm's prompt "
                      f"512 / gen 256: that request takes the oracle ~25-50 min on 8 cores "
                      f"(tests/golden/make_llama8b_bench_golden.py)",
            "same_config": False, "seconds": dt}


GOLDEN = ROOT / "tests" / "golden" / "llama8b_bench_oracle.json"


def measure_traffic(args, timeout_s: int = 240):
    """roofline.traffic: dram__bytes_read.sum + dram__bytes_write.sum of ONE gate/up GEMM launch
    (layer 1 of an un-graphed decode step of this model at batch B, context prompt + gen/2;
    tools/profile_step.py), counted by ncu in a subprocess during this bench run. Byte counts
    only: no time measured under the profiler is reported."""
    import shutil

    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not Path(ncu).exists():
        return None, "ncu not found"
    # GEMM launches per layer: qkv, o, gate/up, down -> the 7th gemm_tc launch is layer 1's gate/up
    cmd = [ncu, "--kernel-name", "regex:gemm_tc_kernel", "--launch-skip", "6", "--launch-count", "1",
           "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum", "--csv", "--clock-control", "none",
           sys.executable, str(ROOT / "tools" / "profile_step.py"), "--model", args.model, "--batch", str(args.batch),
           "--ctx", str(args.prompt + args.gen // 2)]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout_s)
    except (subprocess.TimeoutExpired, OSError) as e:
        return None, f"ncu failed: {str(e)[:120]}"
    vals = {}
    for ln in r.stdout.splitlines():
        parts = [x.strip('"') for x in ln.split('","')]
        if len(parts) >= 3 and parts[-3] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            unit, v = parts[-2], float(parts[-1].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
            vals[parts[-3]] = v * scale
    if len(vals) != 2:
        return None, f"ncu rc={r.returncode}: metrics not found ({(r.stderr or r.stdout)[-160:]!r})"
    return vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"], \
        "ncu (this run, subprocess): gate/up GEMM, layer 1, tools/profile_step.py; read {:.1f} MB + write {:.1f} MB".format(
            vals["dram__bytes_read.sum"] / 1e6, vals["dram__bytes_write.sum"] / 1e6)


def oracle_probes(args, eng, own: dict, rank: int):
    """Compare this run's receipts with the CPU oracle's golden for the same workload. Greedy:
    request 0's hash from the timed workload's e2e leg (rank 0). Nucleus: request 1 re-run with
    p = 0.9 on every rank (all ranks must agree with the oracle)."""
    from paper_2602_00182_b200 import replicas
    from paper_2602_00182_b200.detcore import DecodePolicy

    if not GOLDEN.exists():
        return {"unavailable": "no golden file"}
    g = json.loads(GOLDEN.read_text())
    cases = {c["name"]: c for c in g["cases"]}
    if g["model"] != args.model or any(c["prompt_len"] != args.prompt or c["max_tokens"] != args.gen
                                       for c in cases.values()):
        return {"unavailable": f"golden is for {g['model']} prompt 512 / gen 256"}
    out = {}
    if "greedy" in cases and 0 in own:
        out["greedy_request0"] = own[0].hex() == cases["greedy"]["out_hash"]
    if "nucleus" in cases:
        c = cases["nucleus"]
        _, _, h = eng.generate([replicas.synthetic_prompt(1, args.prompt, eng.vocab)], [DecodePolicy.nucleus(c["p"], args.gen)],
                               [c["seed"]], batch_size=1, want_logits=False)
        out["nucleus_request1"] = h[0].hex() == c["out_hash"]
    return out


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    vals = []
    meta = None
    for i in range(args.warmup + args.steps):
        r = cpu_oracle_sample(args.model, args.cpu_sample_prompt, args.cpu_sample_gen)
        if i >= args.warmup:
            vals.append(r["value"])
            meta = r
    value = float(np.mean(vals))
    ref_toy = None
    try:   # the reference's own engine (toy model only), compiled from its sources into oracle/_ref
        from oracle import oracle as O
        import ctypes as C

        tok = C.c_uint64()
        dt = O.ref().ref_bench(b"model-a", b"archA", 64, 16, 4000, os.cpu_count() or 1, C.byref(tok))
        ref_toy = {"value": tok.value / dt, "unit": "tok/s", "cores": os.cpu_count(),
                   "sample": "reference detcore::infer ToyModel (V=32, d=16), greedy 64, prompt 16, 4000 requests"}
    except Exception as e:   # noqa: BLE001
        ref_toy = {"unavailable": str(e)[:200]}
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tok/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * meta["seconds"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic prompts, random-init weights (counter-based from model_id)",
            "config": {"workload": f"llama3-8b shape greedy decode, bounded CPU sample: prompt {args.cpu_sample_prompt}"
                                   f" / gen {args.cpu_sample_gen} (GPU arm: prompt 512 / gen 256)", "global_batch": 1,
                       "seq_len": args.cpu_sample_prompt + args.cpu_sample_gen, "parallelism": "cpu threads",
                       "same_config": False},
            "cpu_baseline": {k: meta[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": value, "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "reference_toy_engine": ref_toy}
    print(json.dumps(line), flush=True)


def run_ours(args, rank: int, world: int, local: int):
    import torch

    from paper_2602_00182_b200 import _lib as L
    from paper_2602_00182_b200 import replicas
    from paper_2602_00182_b200.detcore import DecodePolicy, Engine

    torch.cuda.set_device(local)
    ctx = args.prompt + args.gen
    eng = Engine(args.model, "b200", max_batch=args.batch, max_context=ctx, device=local)
    V = eng.vocab
    # this rank's requests (weak scaling: every rank serves `batch` requests per step)
    gidx = [rank * args.batch + i for i in range(args.batch)]
    prompts = [replicas.synthetic_prompt(g, args.prompt, V) for g in gidx]
    pols = [DecodePolicy.greedy(args.gen)] * args.batch
    seeds = [replicas.request_seed(g) for g in gidx]

    def gen_device():
        eng.generate(prompts, pols, seeds, device_only=True)
        return eng.last_stats

    for _ in range(args.warmup):
        gen_device()
    # ---- timed region: inputs resident, outputs stay in HBM
    ext = torch.cuda.ExternalStream(L.lib.detgpu_stream(eng.h), device=local)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    replicas.barrier(local)
    torch.cuda.synchronize()
    launches, dev_ms, prefill_ms, decode_ms, toks = 0, 0.0, 0.0, 0.0, 0
    with ClockSampler(local) as clk:
        ev0.record(ext)
        for _ in range(args.steps):
            st = gen_device()
            launches += st.kernel_launches
            prefill_ms += st.prefill_ms
            decode_ms += st.decode_ms
            toks += st.tokens
        ev1.record(ext)
        torch.cuda.synchronize()
    replicas.barrier(local)
    elapsed_ms = ev0.elapsed_time(ev1)
    t_max = replicas.max_over_ranks(elapsed_ms, local)
    toks_all = replicas.sum_over_ranks(toks, local)
    launches_all = replicas.sum_over_ranks(launches, local)
    value = toks_all / (t_max / 1000.0)
    decode_tok_s = (toks - args.batch * args.steps) / (decode_ms / 1000.0) if decode_ms > 0 else None

    # ---- end to end through the C-ABI with host buffers: prompt H2D, logits+tokens D2H, SHA-256
    # e2e_steps batches of the same requests in ONE call with continuous batching (batch slots =
    # args.batch): a finished request's logits D2H and SHA-256 run on a worker thread while the next
    # request decodes, as a server would run them; the bytes of every request are unchanged.
    # warm-up of this leg (pinned receipt buffers, continuous-batching graphs), untimed like the
    # device leg's warm-up steps
    eng.generate(prompts, pols, seeds, batch_size=args.batch, want_logits=False, want_hash=True, continuous=True)
    replicas.barrier(local)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, _, hs_all = eng.generate(prompts * args.e2e_steps, pols * args.e2e_steps, seeds * args.e2e_steps,
                                batch_size=args.batch, want_logits=False, want_hash=True, continuous=True)
    e2e_s = time.perf_counter() - t0
    st = eng.last_stats
    h2d = st.h2d_bytes + sum(p.nbytes for p in prompts) * args.e2e_steps
    d2h = st.d2h_bytes
    hash_ms = st.hash_ms
    hashes = [hs_all[i * args.batch:(i + 1) * args.batch] for i in range(args.e2e_steps)]
    e2e_max = replicas.max_over_ranks(e2e_s, local)
    e2e_value = replicas.sum_over_ranks(args.gen * args.batch * args.e2e_steps, local) / e2e_max
    replay_rate = float(np.mean([h == hashes[0] for h in hashes]))
    # the same calls with receipt v2 (DETGPU_F_RECEIPT_V2): Merkle roots on the GPU, 32 B per step D2H
    v2_s, v2_d2h, v2_hash_ms, v2_hashes = 0.0, 0, 0.0, []
    eng.generate(prompts, pols, seeds, want_logits=False, want_hash=True, receipt_v2=True)   # warm-up
    for _ in range(args.e2e_steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, _, hs = eng.generate(prompts, pols, seeds, want_logits=False, want_hash=True, receipt_v2=True)
        v2_s += time.perf_counter() - t0
        v2_hashes.append(hs)
        v2_d2h += eng.last_stats.d2h_bytes
        v2_hash_ms += eng.last_stats.hash_ms
    v2_max = replicas.max_over_ranks(v2_s, local)
    e2e_v2 = replicas.sum_over_ranks(args.gen * args.batch * args.e2e_steps, local) / v2_max
    # cross-GPU receipt equality by re-execution: every rank re-runs the requests that rank
    # (rank + 1) mod N served above and the hashes are all-gathered (at N = 1 the "other" rank is
    # this one: a replay). Request identity never depends on the rank (replicas.request_seed).
    own = {g: hashes[0][i] for i, g in enumerate(gidx)}
    nxt = (rank + 1) % world
    gnext = [nxt * args.batch + i for i in range(args.batch)]
    _, _, hn = eng.generate([replicas.synthetic_prompt(g, args.prompt, V) for g in gnext], pols,
                            [replicas.request_seed(g) for g in gnext], batch_size=args.batch, want_logits=False)
    cross = replicas.cross_rank_reexecution(own, dict(zip(gnext, hn)), local)
    # the CPU oracle's output for this exact workload (tests/golden/llama8b_bench_oracle.json):
    # request 0 (greedy, this bench's own request) and request 1 (nucleus p = 0.9)
    oracle_probe = oracle_probes(args, eng, own, rank)

    # ---- roofline: live per-kernel timing of one un-graphed decode step (CUDA events per launch)
    import ctypes as C

    ms = (C.c_float * 8)()
    cnt = (C.c_uint32 * 8)()
    L.check(L.lib.detgpu_profile_decode_step(eng.h, args.batch, args.prompt + args.gen // 2, 3, ms, cnt), eng.h)
    info = eng.info
    cls_ms = {CLASS_NAMES[k]: float(ms[k]) for k in range(8)}
    cls_n = {CLASS_NAMES[k]: int(cnt[k]) for k in range(8)}
    d, F, B = info.d_model, info.ffn, args.batch
    gu_bytes = 2.0 * (2 * F) * d + 2.0 * B * d + 2.0 * B * F     # weights + activations in + act out
    gu_launch_ms = cls_ms["gate_up_gemm"] / max(cls_n["gate_up_gemm"], 1)
    peak, peak_kind = peaks()
    achieved = gu_bytes / (gu_launch_ms / 1000.0) / 1e9
    sb = step_bytes(info, B, args.prompt, args.gen)
    step_ms_profiled = sum(cls_ms.values())
    step_ms_graph = decode_ms / max(1, args.steps * (args.gen - 1))
    # the same kernel INSIDE the CUDA-graph step (PDL pipeline): per-CTA timeline, first dependency
    # release -> last CTA end of each gate/up launch (paper_2602_00182_b200/timeline.py)
    graph_span = None
    try:
        from paper_2602_00182_b200 import timeline

        spans, g_ms, g_us = timeline.graph_step_spans(eng, args.batch, args.prompt + args.gen // 2)
        gu = spans.get("gate_up_gemm", [])
        graph_span = {"gate_up_us_mean": float(np.mean(gu)) if gu else None, "launches": len(gu),
                      "achieved_GBs": gu_bytes / (float(np.mean(gu)) * 1e-6) / 1e9 if gu else None,
                      "traced_step_us": g_us, "graph_ms_per_step": g_ms,
                      "class_share_of_step": {k: round(float(np.sum(v)) / g_us, 4) for k, v in spans.items()}}
    except Exception as e:   # noqa: BLE001
        graph_span = {"unavailable": str(e)[:200]}
    # Primary roofline figure: the kernel's duration INSIDE the timed CUDA-graph pipeline = its share
    # of the traced graph step (per-CTA timeline: dependency release -> last CTA end, summed over
    # the step's launches) x the decode-step time measured with CUDA events over the timed region,
    # per launch. The un-graphed per-launch event timing (every kernel starts cold, no PDL overlap
    # with its predecessor) is kept beside it.
    events_ungraphed = {"achieved": achieved, "frac": achieved / peak, "launch_ms": gu_launch_ms,
                        "what": "one un-graphed decode step, CUDA event after every launch"}
    roof_method = "un-graphed CUDA events (trace unavailable)"
    try:
        share = graph_span["class_share_of_step"]["gate_up_gemm"]
        n_gu = graph_span["launches"]
        if share and n_gu and step_ms_graph:
            gu_launch_ms = share * step_ms_graph / n_gu
            achieved = gu_bytes / (gu_launch_ms / 1000.0) / 1e9
            roof_method = ("in-graph: gate/up share of the traced CUDA-graph step (per-CTA timeline) x the "
                           "decode-step time from CUDA events over the timed region, per launch")
    except (KeyError, TypeError):
        pass
    traffic = None
    traffic_src = None

    if rank != 0:
        return
    if args.traffic == "auto" and world == 1:
        traffic, traffic_src = measure_traffic(args)
    sweep = None
    if args.sweep == "auto" and world == 1:
        try:
            sweep = batch_sweep(args.model, eng)
        except Exception as e:   # noqa: BLE001
            sweep = {"unavailable": str(e)[:200]}
    cpu = None
    if args.cpu_baseline == "auto" and world == 1:
        try:
            cpu = cpu_oracle_sample(args.model, args.cpu_sample_prompt, args.cpu_sample_gen)
            cpu.pop("seconds", None)
        except Exception as e:   # noqa: BLE001
            cpu = {"unavailable": str(e)[:200]}
    line = {
        "metric": METRIC, "value": value, "unit": "tok/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic prompts (numpy seeded), random-init weights counter-generated from model_id",
        "config": {"workload": f"llama3-8b shape, greedy decode, batch {B}/GPU, prompt {args.prompt} / gen {args.gen}",
                   "model": args.model, "global_batch": B * world, "seq_len": args.prompt + args.gen,
                   "parallelism": f"replicas x{world}",
                   "l2": "inputs larger than L2: 16 GB of weights streamed every decode step (L2 126 MB)"},
        "e2e": {"value": e2e_value, "unit": "tok/s", "h2d_bytes_per_step": h2d // max(args.e2e_steps, 1),
                "d2h_bytes_per_step": d2h // max(args.e2e_steps, 1),
                "what": "detgpu_generate (continuous batching, e2e_steps copies of the batch in one call) with host "
                        "prompt buffers; tokens + f32 logits D2H; SHA-256 receipt (worker threads)",
                "hash_ms_per_step": hash_ms / max(args.e2e_steps, 1)},
        "e2e_receipt_v2": {"value": e2e_v2, "unit": "tok/s", "d2h_bytes_per_step": v2_d2h // max(args.e2e_steps, 1),
                           "hash_ms_per_step": v2_hash_ms / max(args.e2e_steps, 1),
                           "replay_match_rate": float(np.mean([h == v2_hashes[0] for h in v2_hashes])),
                           "what": "same calls, DETGPU_F_RECEIPT_V2: per-step Merkle roots of the logits on the "
                                   "GPU (DESIGN.md §3.9); tokens + 32 B/step D2H"},
        "roofline": {"bound": "hbm", "kernel": "gate_up_gemm (tcgen05, SwiGLU epilogue)", "achieved": achieved,
                     "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "traffic_source": traffic_src, "method": roof_method, "events_ungraphed": events_ungraphed,
                     "in_graph": graph_span,
                     "peak_source": peak_kind, "bytes_per_launch": gu_bytes, "launch_ms": gu_launch_ms,
                     "step": {"algorithmic_bytes": sb, "graph_step_ms": step_ms_graph,
                              "achieved_GBs": sb / (step_ms_graph / 1000.0) / 1e9 if step_ms_graph else None,
                              "frac": (sb / (step_ms_graph / 1000.0) / 1e9) / peak if step_ms_graph else None},
                     "per_class_ms": cls_ms, "per_class_launches": cls_n, "profiled_step_ms": step_ms_profiled},
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "gpu_launches": int(launches_all),
        "decode_tok_s": decode_tok_s, "prefill_ms": prefill_ms / args.steps,
        "replay_match_rate": replay_rate, "cross_gpu_receipts_equal": bool(cross["all_equal"]),
        "cross_gpu_reexecution": cross,
        "receipt_probe_out_hash": hashes[0][0].hex(),
        "receipt_probe_matches_oracle": oracle_probe.get("greedy_request0"),
        "oracle_probes": oracle_probe,
        "decode_batch_sweep": sweep,
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    from paper_2602_00182_b200 import replicas

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N` without torchrun: launch the N ranks ourselves (one process per
        # GPU, the same torchrun command the driver uses) and pass rank 0's JSON line through.
        sys.exit(replicas.launch_local(args.gpus, [str(Path(__file__).resolve())] + sys.argv[1:]))
    rank, world, local = replicas.dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        if world > 1:
            replicas.init("gloo")
        run_reference(args, rank, world)
        return
    import torch

    torch.cuda.set_device(local)
    replicas.init("nccl")
    run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
