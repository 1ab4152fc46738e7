"""Benchmark: packed-KV decode attention over the NSNQuant cache on B200.

Headline workload (BASELINE.json configs[1]): LLaMA-3-8B attention shape --
32 q-heads / 8 KV-heads (GQA 4), head_dim 128 -- 2-bit cache, batch 16,
context 32K, one decode step = softmax(q.K^T/sqrt(d)).V for every (batch,
q-head) over the packed pages.  Synthetic N(0,1) keys/values encoded by the
product's own encode kernel; q N(0,1).

metric  packed-KV decode attention GB/s: algorithmic bytes per step (the
        reference bit ledger: 2292 B per 64-token K or V chunk in 2-bit,
        vq.py:328-356, plus q in / out) / device time per step.
value   whole job (all ranks), inputs resident in HBM.
e2e     same metric through the public API (PagedKvCache.attend) with q
        copied host->device and the output device->host inside the timing.

``--impl reference`` times the CPU reference path instead (the C oracle, a
restatement of the reference algorithm, on all host cores) on a bounded
sample of the same workload.

Multi-GPU: one process per GPU (torchrun; ``--gpus N`` re-launches itself
under torch.distributed.run when WORLD_SIZE is unset).  The (batch, kv-head)
units are independent, so there is no collective inside attention; outputs are
all-gathered over NCCL at the end of each step (the serving layout's only
exchange).  c2 runs weak scaling (16 sequences per rank); c4 runs strong
scaling (BASELINE config 4: a global batch of 128 split by
sharding.plan_shards, 128/N sequences per rank).
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

D, R = 128, 64
LEDGER = {2: 2292, 1: 1268}
CONFIGS = {
    # name: (batch per rank (weak) or global batch (strong), n_q_heads,
    #        n_kv_heads, context, bit_mode)
    "c2": (16, 32, 8, 32768, 2),
    "c2_1b": (16, 32, 8, 32768, 1),
    "c1": (1, 32, 8, 4096, 1),
    "c4": (128, 32, 8, 131072, 2),
    # not a BASELINE config: GQA group 8 (LLaMA-3-70B head shape), for coverage
    "c2_g8": (16, 64, 8, 32768, 2),
}
STRONG = {"c4"}  # global batch fixed, split over the ranks


def local_batch(cfg_name: str, world: int) -> int:
    B = CONFIGS[cfg_name][0]
    if cfg_name not in STRONG:
        return B
    if B % world:
        raise SystemExit(f"{cfg_name}: global batch {B} does not split over {world} ranks")
    return B // world


def config_dict(cfg_name: str, world: int) -> dict:
    """The workload description -- identical in both arms (same_config)."""
    B, Hq, Hkv, T, bm = CONFIGS[cfg_name]
    strong = cfg_name in STRONG
    gb = B if strong else B * world
    return {"workload": f"{cfg_name}: global batch {gb}, {Hq}q/{Hkv}kv heads, d128, context {T}, "
                        f"{bm}-bit packed KV decode attention (one step = every q-head of every "
                        f"sequence over the whole packed cache)",
            "global_batch": gb, "seq_len": T, "bit_mode": bm,
            "parallelism": f"{'strong' if strong else 'weak'} batch-sharded x{world}"}


def step_bytes(B, Hq, Hkv, T, bit_mode) -> int:
    """Algorithmic bytes of one decode step: every K and V
    chunk's ledger bytes, the residual rows, q in (fp32) and out (fp32)."""
    n_chunks = T // R
    n_res = T - n_chunks * R
    per_unit = n_chunks * LEDGER[bit_mode] * 2 + n_res * D * 4 * 2
    return B * Hkv * per_unit + B * Hq * D * (4 + 4)


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except Exception:
            pass
    return {"hbm_gbs": 6650.0, "_fallback": True}


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region (NVML
    every millisecond; nvidia-smi every 100 ms when NVML is unavailable)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.source = None
        self._nvml = self._nvml_open()
        self._stop = threading.Event()
        self._t = None

    def _nvml_open(self):
        """NVML handle opened before the timed region (init takes tens of ms)."""
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            bits = (pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap)
            return pynvml, h, mx, bits
        except Exception:
            return None

    def _run_nvml(self) -> bool:
        """Fast path: NVML polled every millisecond, so a timed region of a
        few milliseconds still gets several samples (at least one)."""
        if self._nvml is None:
            return False
        pynvml, h, mx, bits = self._nvml
        self.source = "nvml"
        while True:
            try:
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append([str(sm), str(mx)] + ["Active" if r & b else "Not Active" for b in bits])
            except Exception:
                pass
            if self._stop.wait(0.001):
                break
        return True

    def _run(self):
        if self._run_nvml():
            return
        self.source = "nvidia-smi"
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [x.strip() for x in out.stdout.strip().split(",")]
                if len(parts) == 6:
                    self.samples.append(parts)
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples), "source": self.source}


def dist_setup():
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(local)
    return world, rank, local


def build_cache(cfg_name: str, device, seed: int, precision: str | None = None, world: int = 1):
    """Encode a synthetic cache of the workload shape (this rank's share)
    with the product's own append path (chunked so staging stays small)."""
    import torch

    import paper_2505_18231_b200 as P

    _, Hq, Hkv, T, bm = CONFIGS[cfg_name]
    B = local_batch(cfg_name, world)
    cb = P.default_codebook(f"{bm}b")
    cfg = P.CacheConfig(d=D, bit_mode=cb.bit_mode)
    cache = P.PagedKvCache(cfg, B, Hkv, max_tokens=T, cb_k=cb, cb_v=cb, device=device,
                           check_finite=False, precision=precision)
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    block = max(R, min(4096, (1 << 26) // (B * Hkv * D) // R * R))
    done = 0
    while done < T:
        n = min(block, T - done)
        k = torch.randn(B, Hkv, n, D, device=device, generator=gen, dtype=torch.bfloat16)
        v = torch.randn(B, Hkv, n, D, device=device, generator=gen, dtype=torch.bfloat16)
        cache.append(k, v)
        done += n
    torch.cuda.synchronize()
    return cache


def time_attend(cache, q, out, steps: int) -> float:
    """ms per nsnkv_decode_attend call (CUDA events on the launching stream,
    warm-up first)."""
    import torch

    for _ in range(3):
        cache.attend(q, out=out)
    torch.cuda.synchronize()
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k0.record()
    for _ in range(steps):
        cache.attend(q, out=out)
    k1.record()
    torch.cuda.synchronize()
    return k0.elapsed_time(k1) / steps


def run_ours(args) -> dict | None:
    import torch

    import paper_2505_18231_b200 as P

    world, rank, local = dist_setup()
    device = torch.device("cuda", local)
    _, Hq, Hkv, T, bm = CONFIGS[args.config]
    B = local_batch(args.config, world)
    cache = build_cache(args.config, device, seed=1234 + rank, precision=args.precision,
                        world=world)
    gen = torch.Generator(device=device)
    gen.manual_seed(99 + rank)
    q = torch.randn(B, Hq, D, device=device, generator=gen)
    out = torch.empty(B, Hq, D, device=device)
    # each rank owns a contiguous batch range (paper_2505_18231_b200.sharding);
    # one all-gather of outputs per step into a pre-allocated buffer
    from paper_2505_18231_b200.sharding import gather_buffer, gather_outputs, plan_shards

    gb = B * world
    plan = plan_shards(gb, Hkv, Hq, world, rank)
    gbuf = gather_buffer(plan, out) if world > 1 else None

    def step():
        cache.attend(q, out=out)
        if world > 1:
            gather_outputs(plan, out, buf=gbuf)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    launches0 = P._lib.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    launches = P._lib.launch_count() - launches0
    ms = e0.elapsed_time(e1) / args.steps
    t_max = torch.tensor([ms], device=device)
    if world > 1:
        torch.distributed.all_reduce(t_max, op=torch.distributed.ReduceOp.MAX)
    ms = float(t_max.item())
    sbytes = step_bytes(B, Hq, Hkv, T, bm)
    value = sbytes * world / (ms * 1e-3) / 1e9

    # dominant kernel: the attend launch alone (CUDA events on its stream)
    k_ms = time_attend(cache, q, out, args.steps)

    # e2e through the public API: every step uploads its q from pinned host
    # memory, runs PagedKvCache.attend (+ the output all-gather when sharded)
    # and downloads its output to pinned host memory.  The copies run on a
    # second stream, double-buffered: step i+1's upload and step i's download
    # overlap step i's / i+1's kernels, as a serving loop would run them.
    q_host = q.cpu().pin_memory()
    out_host = [torch.empty(B, Hq, D).pin_memory() for _ in range(2)]
    q_dev = [torch.empty_like(q) for _ in range(2)]
    out_dev = [torch.empty_like(out) for _ in range(2)]
    main, side = torch.cuda.current_stream(), torch.cuda.Stream()
    up = [torch.cuda.Event() for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]

    def e2e_steps(n):
        with torch.cuda.stream(side):
            q_dev[0].copy_(q_host, non_blocking=True)
            up[0].record(side)
        for i in range(n):
            cur, nxt = i % 2, (i + 1) % 2
            main.wait_event(up[cur])
            cache.attend(q_dev[cur], out=out_dev[cur])
            if world > 1:
                gather_outputs(plan, out_dev[cur], buf=gbuf)
            done[cur].record(main)
            with torch.cuda.stream(side):
                if i + 1 < n:
                    if i >= 1:
                        side.wait_event(done[nxt])  # step i-1 is done with q_dev[nxt]
                    q_dev[nxt].copy_(q_host, non_blocking=True)
                    up[nxt].record(side)
                side.wait_event(done[cur])
                out_host[cur].copy_(out_dev[cur], non_blocking=True)
        main.wait_stream(side)

    e2e_steps(3)
    torch.cuda.synchronize()
    barrier()
    x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    x0.record()
    e2e_steps(args.steps)
    x1.record()
    torch.cuda.synchronize()
    e2e_ms = x0.elapsed_time(x1) / args.steps
    t2 = torch.tensor([e2e_ms], device=device)
    if world > 1:
        torch.distributed.all_reduce(t2, op=torch.distributed.ReduceOp.MAX)
    e2e_ms = float(t2.item())

    peaks = measured_peaks()
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = sbytes / (k_ms * 1e-3) / 1e9
    if rank != 0:
        return None
    traffic = None
    tp = ROOT / "profiles" / "traffic.json"
    if tp.exists():
        try:
            traffic = json.loads(tp.read_text()).get(f"{args.config}:{cache.precision}")
        except Exception:
            traffic = None
    res = {
        "metric": "packed-KV decode attention GB/s",
        "value": round(value, 2),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 4),
        "higher_is_better": True,
        "scaling": "strong" if args.config in STRONG else "weak",
        "vs_baseline": None,
        "dtype": "u8 pages / fp32 accumulate",
        "data": "synthetic N(0,1) K/V (bf16) encoded by the product; N(0,1) q",
        "config": {**config_dict(args.config, world),
                   "l2": "inputs larger than L2 (packed cache %.0f MB/rank)" % (sbytes / 1e6)},
        "precision": cache.precision,
        "tokens_per_s": round(gb / (ms * 1e-3), 1),
        "e2e": {"value": round(sbytes * world / (e2e_ms * 1e-3) / 1e9, 2), "unit": "GB/s",
                "h2d_bytes_per_step": B * Hq * D * 4, "d2h_bytes_per_step": B * Hq * D * 4,
                "ms_per_step": round(e2e_ms, 4),
                "how": "PagedKvCache.attend per step; q pinned-host -> device and out device -> "
                       "pinned-host every step on a copy stream, double-buffered"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if not peaks.get("_fallback")
                     else "fallback 6.65 TB/s (B200_PROFILING.md)",
                     "kernel": "nsnkv_decode_attend", "kernel_ms": round(k_ms, 4),
                     "bytes_per_launch": sbytes},
        "clocks": clk.summary(),
        "gpu_launches": int(launches),
    }
    if world == 1 and not args.no_extras:
        extras = {}
        if args.config == "c2":
            # the like-for-like all-hi+lo mode on the same cache
            prev = cache.precision
            cache.precision = "precise"
            extras["c2_precise"] = kernel_line(sbytes, time_attend(cache, q, out, args.steps), peak)
            cache.precision = prev
        res["serving_step"] = measure_serving(cache, q, steps=2 * R)
        del cache
        torch.cuda.empty_cache()
        if args.config == "c2":
            for name in ("c2_1b", "c4", "c2_g8"):
                extras[name] = measure_config(name, device, peak, steps=max(10, args.steps // 5))
        res["extras"] = extras
        res["encode"] = {f"{m}b": measure_encode(device, m) for m in (2, 1)}
        if args.config == "c2" and not args.no_model:
            res["c5_model"] = measure_c5(device)
        res["parity"] = c1_parity()
    if world == 1 and not args.no_cpu_baseline:
        res["cpu_baseline"] = cpu_baseline(args.config, budget_s=args.cpu_budget)
    return res


def measure_c5(device) -> dict:
    """BASELINE config 5 per GPU: full LLaMA-3.1-8B-shape random-init decode
    step, batch 32 x 16K (the per-GPU share of batch 256 on 8 GPUs, DP=8),
    NSNQuant 1-bit KV (fused decode_step) vs bf16 KV (flash-attn)."""
    sys.path.insert(0, str(ROOT / "scripts"))
    import bench_model as BM

    out = {}
    for kv in ("nsn1b", "bf16"):
        out[kv] = BM.run(kv, 32, 16384, 32, steps=6, warmup=2, dev=device)
    out["speedup_vs_bf16"] = round(out["nsn1b"]["tokens_per_s_job"] / out["bf16"]["tokens_per_s_job"], 3)
    return out


def kernel_line(sbytes: int, ms: float, peak: float) -> dict:
    gbs = sbytes / (ms * 1e-3) / 1e9
    return {"ms": round(ms, 4), "GBps": round(gbs, 1), "frac": round(gbs / peak, 4)}


def measure_config(name: str, device, peak: float, steps: int) -> dict:
    """One more BASELINE workload on this GPU (default precision)."""
    import torch

    _, Hq, Hkv, T, bm = CONFIGS[name]
    B = local_batch(name, 1)
    cache = build_cache(name, device, seed=4321)
    q = torch.randn(B, Hq, D, device=device)
    out = torch.empty(B, Hq, D, device=device)
    sb = step_bytes(B, Hq, Hkv, T, bm)
    line = kernel_line(sb, time_attend(cache, q, out, steps), peak)
    line.update({"workload": config_dict(name, 1)["workload"], "precision": cache.precision,
                 "tokens_per_s": round(B / (line["ms"] * 1e-3), 1)})
    del cache
    torch.cuda.empty_cache()
    return line


def c1_parity() -> dict:
    """Counted differences of the GPU's pages against the REFERENCE's own
    serialized chunks on BASELINE config 1 (tests/golden/c1_*.npz, made by
    tests/golden/gen_c1.py), and the decode error against its outputs."""
    import torch

    import paper_2505_18231_b200 as P
    from tests.golden.inputs import c1_inputs, c1_value_entries
    from tests.parity_bounds import summarize
    from tests.wirediff import compare

    counts, worst = [], 0.0
    for case in c1_inputs():
        with np.load(ROOT / "tests" / "golden" / f"c1_{case['name']}.npz") as z:
            g = {k: z[k] for k in ("k_wire", "v_wire", "out")}
        cb_k = P.default_codebook(f"{case['bit_mode']}b")
        cb_v = cb_k if not case["distinct_v"] else P.Codebook(
            entries=c1_value_entries(cb_k.entries, True), bit_mode=cb_k.bit_mode)
        H = case["keys"].shape[0]
        c = P.PagedKvCache(P.CacheConfig(d=D, bit_mode=cb_k.bit_mode), 1, H, cb_k=cb_k, cb_v=cb_v)
        k = torch.from_numpy(case["keys"][None]).cuda()
        v = torch.from_numpy(case["values_ht"][None]).cuda()
        for a, b in case["batches"]:
            c.append(k[:, :, a:b], v[:, :, a:b])
        for kind in ("k", "v"):
            got = np.stack([c.wire_chunks(u, kind) for u in range(H)])
            counts.append(compare(got, g[f"{kind}_wire"], case["bit_mode"]))
        out = c.attend(torch.from_numpy(case["q"].reshape(1, -1, D)).cuda()).cpu().numpy()
        out = out.reshape(g["out"].shape)
        err = np.abs(out - g["out"]).max(axis=-1) / np.abs(g["out"]).max(axis=-1)
        worst = max(worst, float(err.max()))
    tot = summarize(counts)
    tot["decode_max_rel_err"] = float(f"{worst:.3g}")
    tot["what"] = ("BASELINE config 1 (8 KV heads x 4133 tokens, 1b/2b, N(0,1)/misaligned) vs the "
                   "reference's serialized chunks and attend_quantized outputs")
    return tot


def measure_serving(cache, q, steps: int) -> dict:
    """One decode step as a server runs it (PagedKvCache.decode_step): append
    this step's K/V token for every (sequence, kv-head) and attend over the
    cache including it -- in the attend launches when no chunk completes, a
    64-token chunk flushed through nsnkv_append every 64 steps.  Averaged
    over `steps` steps (a multiple of 64, so the flushes are included)."""
    import torch

    B, Hkv = cache.batch, cache.n_kv_heads
    dev = q.device
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    ks = torch.randn(steps, B, Hkv, 1, D, device=dev, generator=g)
    vs = torch.randn(steps, B, Hkv, 1, D, device=dev, generator=g)
    out = torch.empty_like(q)
    cache.reserve(cache.total_tokens + steps)  # pools sized up front, as a server does
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(steps):
        cache.decode_step(q, ks[i], vs[i], out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    return {"what": "PagedKvCache.decode_step: append 1 token/sequence (flush every 64) + attend",
            "ms_per_step": round(ms, 4),
            "tokens_per_s": round(B / (ms * 1e-3), 1), "steps": steps,
            "context_after": cache.total_tokens}


def measure_encode(device, bit_mode: int, batch: int = 64, heads: int = 8, tokens: int = 8192) -> dict:
    """BASELINE config 3: prefill quantize/append of a 64 x 8K x 8-head
    bf16 K/V batch (one append call, all chunks flushed)."""
    import torch

    import paper_2505_18231_b200 as P

    cb = P.default_codebook(f"{bit_mode}b")
    cfg = P.CacheConfig(d=D, bit_mode=cb.bit_mode)
    g = torch.Generator(device=device)
    g.manual_seed(3)
    k = torch.randn(batch, heads, tokens, D, device=device, generator=g).to(torch.bfloat16)
    v = torch.randn(batch, heads, tokens, D, device=device, generator=g).to(torch.bfloat16)
    times = []
    for it in range(3):
        cache = P.PagedKvCache(cfg, batch, heads, max_tokens=tokens, cb_k=cb, cb_v=cb,
                               device=device, check_finite=False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        cache.append(k, v)
        e1.record()
        torch.cuda.synchronize()
        if it:
            times.append(e0.elapsed_time(e1))
    ms = min(times)
    th = batch * heads * tokens
    nbytes = th * D * 2 * 2 + (th // R) * LEDGER[bit_mode] * 2
    macs = th * 2 * 16 * 256 * 8
    del k, v, cache
    torch.cuda.empty_cache()
    return {"workload": f"config 3: batch {batch} x {heads} kv-heads x {tokens} tokens, bf16 in, "
                        f"{bit_mode}-bit", "ms": round(ms, 3),
            "token_heads_per_s": round(th / (ms * 1e-3), 1),
            "GBps_algorithmic": round(nbytes / (ms * 1e-3) / 1e9, 1),
            "search_TMACps": round(macs / (ms * 1e-3) / 1e12, 2),
            "bound": "compute (codebook search, 32768 MAC per token vector)"}


_CPU_SAMPLE = {}


def cpu_baseline(cfg_name: str, budget_s: float = 15.0, threads: int | None = None) -> dict:
    """The oracle (C restatement of the reference path) on the host cores:
    encode one full-context (batch, kv-head) unit once, replicate it over one
    unit per host thread, then time attend_quantized-equivalent decode of all
    G q-heads of every unit, repeated until `budget_s` of CPU work."""
    from oracle import oracle as orc

    B, Hq, Hkv, T, bm = CONFIGS[cfg_name]
    G = Hq // Hkv
    cores = threads or os.cpu_count() or 1
    # the shipped codebook read by the oracle's own NSNC reader: this arm
    # never loads the product package or its CUDA library
    ent, _ = orc.load_nsnc_entries(ROOT / "paper_2505_18231_b200" / "codebooks" / f"cb{bm}_seed0.nsnc")
    n_chunks = T // R
    key = (cfg_name, cores)
    if key not in _CPU_SAMPLE:
        # one unit's pages, replicated across the sample (decode cost is
        # data-independent); encoded by the oracle itself
        g = np.random.Generator(np.random.PCG64(7))
        k = g.standard_normal((n_chunks, R, D), dtype=np.float32)
        v = g.standard_normal((n_chunks, R, D), dtype=np.float32)
        kw = orc.encode_many(k, True, ent, bm, threads=cores)  # keys at pos 0 per chunk
        vw = orc.encode_many(v, False, ent, bm, threads=cores)
        kws = np.ascontiguousarray(np.broadcast_to(kw.reshape(1, -1), (cores, kw.size)))
        vws = np.ascontiguousarray(np.broadcast_to(vw.reshape(1, -1), (cores, vw.size)))
        q = g.standard_normal((cores, G, D), dtype=np.float32)
        _CPU_SAMPLE[key] = (kws, vws, q)
    kws, vws, q = _CPU_SAMPLE[key]
    n_units = cores
    reps, t0 = 0, time.perf_counter()
    while True:
        orc.attend_many(kws, vws, n_units, n_chunks, ent, ent, bm, q, threads=cores)
        reps += 1
        dt = time.perf_counter() - t0
        if dt >= budget_s:
            break
    unit_bytes = n_chunks * LEDGER[bm] * 2 + G * D * 8
    return {"value": round(reps * n_units * unit_bytes / dt / 1e9, 4), "unit": "GB/s", "cores": cores,
            "kind": "port",
            "sample": f"{reps} x {n_units} full-context units x {G} q-heads ({T} tokens, {bm}-bit) "
                      f"decoded in {dt:.2f}s on {cores} threads; extrapolated to the workload "
                      f"({B * Hkv} units per rank): the per-unit decode cost is data-independent, "
                      f"so GB/s does not depend on the unit count",
            "extrapolated": True,
            "seconds": round(dt, 3)}


def run_reference(args) -> dict | None:
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    vals = []
    # seconds of CPU work per step: 3 s, less when many steps are asked for so
    # the whole run stays within ~2.5 minutes
    step_budget = float(os.environ.get("NSNKV_REF_STEP_S", "3"))
    step_budget = max(0.2, min(step_budget, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        cpu_baseline(args.config, budget_s=step_budget)
    for _ in range(args.steps):
        vals.append(cpu_baseline(args.config, budget_s=step_budget))
    best = vals[-1]
    value = float(np.median([v["value"] for v in vals]))
    return {
        "impl": "reference", "metric": "packed-KV decode attention GB/s", "value": value,
        "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "higher_is_better": True, "scaling": "strong" if args.config in STRONG else "weak",
        "vs_baseline": None, "dtype": "u8 pages / fp32 accumulate", "data": "synthetic N(0,1)",
        "config": config_dict(args.config, world),
        "cpu_baseline": {**best, "value": value},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the serving-step and encode measurements")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-model", action="store_true", help="skip the C5 full-model extra")
    ap.add_argument("--precision", default=None, choices=["precise", "vfast"],
                    help="decode codeword precision (DESIGN.md 3.2); default: the library's "
                         "(vfast for 2-bit, precise for 1-bit)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
               str(Path(__file__).resolve()), *sys.argv[1:]]
        raise SystemExit(subprocess.run(cmd).returncode)
    res = run_reference(args) if args.impl == "reference" else run_ours(args)
    if res is not None:
        print(json.dumps(res), flush=True)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1 and args.impl != "reference":
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
