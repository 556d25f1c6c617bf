#!/usr/bin/env python3
"""bench.py -- the FP8 W8A8 rollout hot path (arXiv 2601.18150 §2.1) on B200.

Headline (BASELINE.json configs[1], the config the metric is quoted on): one Qwen3-8B
transformer layer's linear layers at prefill M = 8192 tokens per GPU.  One STEP = one pass of
the whole hot path:
  1. weight sync: blockwise requantization of the layer's four BF16 weights
     (qkv 6144x4096, o 4096x4096, gate_up 24576x4096, down 4096x12288) -- sharded by
     128-row blocks over the N ranks, then an in-place NCCL all-gather of the FP8 codes and
     scales (N > 1 only);
  2. dynamic per-token-group activation quantization of the four GEMM inputs;
  3. the four blockwise-scaled FP8 GEMMs, BF16 output.
metric = GEMM TFLOP/s of the whole step (all ranks' GEMM FLOPs / max-over-ranks step time);
requant GB/s, activation-quant GB/s and GEMM-only TFLOP/s are reported alongside.

The same JSON line carries the other §8(d) rows as sub-records (each with absolute numbers,
its roofline and the clocks of its window): `decode` (configs[2], M = 1/64/128/256, one CUDA
graph per layer: 4 activation quantizations + 4 GEMMs), `moe` (configs[3], Qwen3-30B-A3B
experts, T = 1024 / 8192, uniform and Zipf routing, plus the EP-8 shard), `sync` (configs[4],
whole-model Qwen3-8B and Qwen3-30B-A3B requant at P = world) and `tp_shards` (the
column-parallel GEMM shards of north_star at P = 2/4/8).

Timing (B200_PROFILING.md): W untimed warm-up steps; K timed steps, each bracketed by CUDA
events on the launching stream; no L2 flush for the headline step: its inputs are larger
than L2 (each step reads ~0.79 GB of BF16 weights and activations and writes ~0.64 GB, every
tensor once); sub-records either flush L2 (a 256 MB write) before every timed launch or rotate
over weight copies larger than L2 (decode graphs), as each says; barrier + synchronize on
both sides; max over ranks; nvidia-smi clocks sampled throughout.  `e2e` repeats the headline
step through the same C-ABI calls with HOST (pinned) inputs: H2D of the step's BF16 weight
shards and activations and D2H of the GEMM outputs are inside its timed region.

--gpus N (N > 1) without a torchrun environment relaunches itself under
`torch.distributed.run` with N ranks (NCCL_DEBUG=INFO so the communicator lines show N ranks).
--impl reference times the CPU oracle (the reference arm of this tier; deliberately slow) on
a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402

METRIC = "blockwise-FP8 GEMM TFLOP/s (Qwen3-8B shapes); weight requant GB/s vs HBM"
WORKLOAD = "qwen3_8b_layer_linears_prefill_m8192"
M_PREFILL = 8192
WEIGHT_BYTES_PER_ELEM = 3.0 + 4.0 / 16384  # 2 B read + 1 B code + 4 B scale per 128x128
ACT_BYTES_PER_ELEM = 3.0 + 4.0 / 128
PAPER_CONTEXT = ("PAPER.md:16,193: up to 44% rollout-throughput speedup for Qwen3-8B with FP8 linear layers + "
                 "FP8 KV cache (+ attention) vs BF16, on 8xH100 (vLLM/SGLang + DeepGEMM); context only, not a "
                 "kernel-level target")


# ----------------------------------------------------------------------------- helpers
def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return {"hbm_gbs": float(p["hbm_gbs"]), "bf16_tflops": float(p["bf16_tflops"]),
                "bf16_tflops_sustained": float(p.get("bf16_tflops_sustained", p["bf16_tflops"])),
                "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "source": "fallback (B200_PROFILING.md)"}


def fp8_peak_tflops(peaks, sustained=True):
    """FP8 dense = 2x BF16 dense (nominal 4.5 / 2.25 PFLOP/s) applied to the measured cuBLAS BF16
    peak.  The headline step runs after >= 1.5 s of warm-up, i.e. in the power-capped steady
    state, so its denominator is the SUSTAINED figure; kernels timed alone (sub-records) use
    the burst one (B200_PROFILING.md)."""
    return 2.0 * (peaks["bf16_tflops_sustained"] if sustained else peaks["bf16_tflops"])


class ClockSampler:
    """nvidia-smi clocks/throttle reasons at 200 ms for the whole run; `summary(t0, t1)` gives the
    samples of one window (host perf_counter times)."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["active_mask", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device_index: int):
        p = torch.cuda.get_device_properties(device_index)
        self.gpu = f"{p.pci_domain_id:08X}:{p.pci_bus_id:02X}:{p.pci_device_id:02X}.0"
        self.proc = None
        self.rows = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", self.gpu, f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.strip().split(",")]
            if len(parts) < 8:
                continue
            try:
                self.rows.append((time.perf_counter(), float(parts[0]), float(parts[1]), float(parts[2]), parts[3:]))
            except ValueError:
                continue

    def summary(self, t0=None, t1=None):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = [r for r in self.rows if (t0 is None or r[0] >= t0 - 0.2) and (t1 is None or r[0] <= t1 + 0.2)]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples in window"]}
        loaded = [r for r in rows if r[3] > 250.0] or rows
        reasons = sorted({self.NAMES[i] for r in loaded for i, v in enumerate(r[4]) if i > 0 and v == "Active"})
        return {"sm_mhz": float(np.median([r[1] for r in loaded])), "sm_max_mhz": max(r[2] for r in rows),
                "reasons": reasons, "samples": len(rows), "samples_under_load": len(loaded),
                "power_w_max": max(r[3] for r in rows)}

    def stop(self):
        time.sleep(0.25)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def init_dist(world, local):
    device = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(device)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=device)
    return device


def max_over_ranks(x: float, device, world) -> float:
    t = torch.tensor([x], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class L2Flush:
    """Between timed launches: write a 256 MB buffer (> 126 MB L2), then read it back, so every
    timed kernel starts with a cold L2 that holds other, CLEAN data.  (A write alone leaves
    ~126 MB of dirty lines whose write-back the next kernel pays: ~20 us, which dominated the
    small shard / expert GEMMs in the first round-2 bench line.)"""

    def __init__(self, device):
        self.buf = torch.empty(256 << 20, dtype=torch.uint8, device=device)

    def __call__(self):
        self.buf.zero_()
        self.buf.view(torch.int64).sum()


def time_launch(fn, flush: L2Flush, iters: int = 10, warm: int = 2) -> float:
    """Median ms of `fn` over `iters` launches, each after an L2 flush, bracketed by CUDA events
    on the current stream (the GPU is kept busy while the host enqueues, so launch overhead of
    the binding is not timed)."""
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(iters):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(300_000)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def bf16_from_bits(bits: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16)


def dev_bf16(shape, gen, device, std=1.0):
    """Device-generated seeded BF16 (bench data only; parity inputs come from synth/)."""
    t = torch.empty(shape, dtype=torch.bfloat16, device=device)
    flat = t.view(-1)
    for c0 in range(0, flat.numel(), 1 << 26):
        c1 = min(flat.numel(), c0 + (1 << 26))
        flat[c0:c1] = (torch.randn(c1 - c0, generator=gen, device=device) * std).to(torch.bfloat16)
    return t


# ----------------------------------------------------------------------------- headline step
LAYER = [("qkv",) + synth.QWEN3_8B_LINEARS["qkv"], ("o",) + synth.QWEN3_8B_LINEARS["o"],
         ("gate_up",) + synth.QWEN3_8B_LINEARS["gate_up"], ("down",) + synth.QWEN3_8B_LINEARS["down"]]


# e2e upload / GEMM / read-back order: H2D and D2H share ~98 GB/s of PCIe when both run, so the
# GEMM with the largest output goes first (a PCIe model of the four orders puts this one 4 %
# ahead of qkv-first: 18.2 vs 19.0 ms)
E2E_ORDER = [LAYER[2], LAYER[3], LAYER[1], LAYER[0]]  # gate_up, down, o, qkv
# activation upload / GEMM / read-back row blocks per GEMM (the same PCIe model: 19.0 -> 17.0 ms
# at 4 blocks; the GEMMs run on 2,048-row blocks, hidden behind the transfers)
E2E_CHUNKS = int(os.environ.get("FP8Q_E2E_CHUNKS", "4"))  # row blocks per GEMM in the e2e pipeline (env: dev A/B)


def layer_flops(m):
    return sum(2.0 * m * n * k for _, n, k in LAYER)


def headline_config(world, m=M_PREFILL):
    """The config dict both arms print (same keys, same values)."""
    return {"workload": WORKLOAD, "tokens_per_gpu": m, "global_batch": m * world,
            "gemms": {n: [m, nn, k] for n, nn, k in LAYER}, "out_dtype": "bf16",
            "l2": "inputs larger than L2 (0.79 GB read + 0.64 GB written per step vs 126 MB L2; no flush)",
            "parallelism": f"dp{world}: per-step weight requant sharded by 128-row blocks"
                           + (" + NCCL all-gather of FP8 codes/scales" if world > 1 else "")}


class LayerStep:
    """Device buffers and the step of the headline workload on one rank."""

    def __init__(self, world, rank, device, m=M_PREFILL):
        from paper_2601_18150_b200 import fp8q
        from paper_2601_18150_b200.sync import TensorSpec, WeightSyncEngine
        self.fp8q = fp8q
        self.m = m
        self.device = device
        self.world = world
        # the e2e pipeline's order (the sync walks its specs in this order): gate_up (largest
        # output) first, so its 403 MB read-back overlaps the remaining uploads
        specs = [TensorSpec(name, n, k) for name, n, k in E2E_ORDER]
        self.engine = WeightSyncEngine(specs, device)
        # host (pinned) BF16 weight shards and activations, from the seeded generators
        self.h_w, self.h_x = {}, {}
        for i, (name, n, k) in enumerate(LAYER):
            r0, r1 = self.engine.shard_rows(name)
            full = synth.qwen3_weight(n, k, seed=i)
            self.h_w[name] = bf16_from_bits(full[r0:r1]).pin_memory()
            self.h_x[name] = bf16_from_bits(synth.qwen3_activation(m, k, seed=100 * rank + i)).pin_memory()
        self.w = {k: v.to(device) for k, v in self.h_w.items()}
        self.x = {k: v.to(device) for k, v in self.h_x.items()}
        self.xq, self.xs, self.y = {}, {}, {}
        for name, n, k in LAYER:
            self.xq[name] = torch.empty((m, k), dtype=torch.uint8, device=device)
            self.xs[name] = torch.empty((k // 128, fp8q.act_scales_ld(m)), dtype=torch.float32, device=device)
            self.y[name] = torch.empty((m, n), dtype=torch.bfloat16, device=device)
        self.h_y = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True) for k, v in self.y.items()}
        self.comm = torch.cuda.Stream(device) if world > 1 else None
        self.step_id = 0
        self.weight_elems_local = sum(v.numel() for v in self.w.values())
        self.act_elems = sum(v.numel() for v in self.x.values())

    def run(self, ev=None):
        fq = self.fp8q
        self.step_id += 1
        # strict=False: the non-finite flag is checked after the timed region (no host sync here)
        self.engine.sync_step(self.step_id, self.w, self.comm, strict=False)
        if ev:
            ev[1].record()
        # the layer's four GEMM inputs in one persistent launch
        fq.quantize_act_per_token_group_batched([(self.x[nm], self.xq[nm], self.xs[nm]) for nm, _, _ in LAYER])
        if ev:
            ev[2].record()
        for name, _, _ in LAYER:
            fq.fp8_block_gemm(self.xq[name], self.xs[name], self.engine.codes[name], self.engine.scales[name],
                              out=self.y[name])

    def run_e2e(self, chunks: int = E2E_CHUNKS):
        """The step through the same C-ABI calls with host (pinned) inputs and outputs, as a
        pipeline over four streams in E2E_ORDER (gate_up first): H2D uploads each GEMM's weight
        shard, then its activations in `chunks` row blocks; the weight sync quantizes (and
        gathers) each tensor as soon as its shard has landed (buckets of one tensor); the
        activation quantization + GEMM of each row block runs on a GEMM stream as soon as the
        block and the FP8 weight are there; D2H reads each output row block back as soon as it
        is produced (so the read-back of the first blocks overlaps the remaining uploads)."""
        fq = self.fp8q
        cur = torch.cuda.current_stream(self.device)
        if not hasattr(self, "_h2d"):
            self._h2d = torch.cuda.Stream(self.device)
            self._d2h = torch.cuda.Stream(self.device)
            self._gs = torch.cuda.Stream(self.device)
        h2d, d2h, gs = self._h2d, self._d2h, self._gs
        h2d.wait_stream(cur)
        gs.wait_stream(cur)
        m = self.m
        bounds = [m * c // chunks for c in range(chunks + 1)]
        ev_w, ev_x, ev_q = {}, {}, {}
        with torch.cuda.stream(h2d):
            for name, _, _ in E2E_ORDER:
                self.w[name].copy_(self.h_w[name], non_blocking=True)
                ev_w[name] = torch.cuda.Event()
                ev_w[name].record(h2d)
                for c in range(chunks):
                    r0, r1 = bounds[c], bounds[c + 1]
                    self.x[name][r0:r1].copy_(self.h_x[name][r0:r1], non_blocking=True)
                    ev_x[(name, c)] = torch.cuda.Event()
                    ev_x[(name, c)].record(h2d)

        def quantized(names):
            for nm in names:
                ev_q[nm] = torch.cuda.Event()
                ev_q[nm].record(torch.cuda.current_stream(self.device))

        self.step_id += 1
        self.engine.sync_step(self.step_id, self.w, self.comm, bucket=1, ready=ev_w, on_bucket=quantized,
                              strict=False)
        for name, _, _ in E2E_ORDER:
            for c in range(chunks):
                r0, r1 = bounds[c], bounds[c + 1]
                with torch.cuda.stream(gs):
                    gs.wait_event(ev_x[(name, c)])
                    if c == 0:
                        gs.wait_event(ev_q[name])
                    xq, xs = self.xq[name][r0:r1], self.xs[name][:, r0:r1]
                    fq.quantize_act_per_token_group(self.x[name][r0:r1], xq, xs)
                    fq.fp8_block_gemm(xq, xs, self.engine.codes[name], self.engine.scales[name],
                                      out=self.y[name][r0:r1])
                    ev_y = torch.cuda.Event()
                    ev_y.record(gs)
                d2h.wait_event(ev_y)
                with torch.cuda.stream(d2h):
                    self.h_y[name][r0:r1].copy_(self.y[name][r0:r1], non_blocking=True)
        cur.wait_stream(gs)
        cur.wait_stream(d2h)
        cur.wait_stream(h2d)

    def h2d_bytes(self):
        return sum(v.numel() * 2 for v in self.h_w.values()) + sum(v.numel() * 2 for v in self.h_x.values())

    def d2h_bytes(self):
        return sum(v.numel() * 2 for v in self.h_y.values())


# ----------------------------------------------------------------------------- sub-records
def decode_layer_bytes(m):
    """Algorithmic HBM bytes of one decode layer: per GEMM
    N*K + M*K + 4*(M*K/128 + N*K/16384) + 2*M*N, plus the four activation quantizations
    (2 B read + 1 B + 4 B/128 written per element; their 1 B codes are the GEMM's M*K)."""
    by = 0.0
    for _, n, k in LAYER:
        by += n * k + m * k + 4.0 * (m * k / 128 + n * k / 16384) + 2.0 * m * n
        by += m * k * (2.0 + 4.0 / 128)
    return by


def bench_decode(st: LayerStep, peaks, clocks, ms=(1, 64, 128, 256), copies=4, replays=8):
    """C3 (BASELINE.json configs[2]): one Qwen3-8B decode layer = 4 activation quantizations +
    4 GEMMs, captured as ONE CUDA graph per layer; the graph walks `copies` distinct copies of
    the layer's FP8 weights (4 x 193 MB > L2), so every layer streams its weights from HBM."""
    fq = st.fp8q
    dev = st.device
    layers = [(st.engine.codes, st.engine.scales)]
    for _ in range(copies - 1):
        layers.append(({k: v.clone() for k, v in st.engine.codes.items()},
                       {k: v.clone() for k, v in st.engine.scales.items()}))
    out = {}
    t_win = time.perf_counter()
    for m in ms:
        xs = {nm: st.x[nm][:m] for nm, _, _ in LAYER}
        ys = {nm: torch.empty((m, n), dtype=torch.bfloat16, device=dev) for nm, n, _ in LAYER}

        def layer(c, s, which=None):
            # each linear as the rollout engine calls it: BF16 input, dynamic activation
            # quantization + blockwise FP8 GEMM, chained by programmatic dependent launch)
            for nm, _, _ in LAYER:
                if which is None or nm == which:
                    fq.fp8_linear_dynamic(xs[nm], c[nm], s[nm], out=ys[nm])

        def graph_us(which=None):
            s = torch.cuda.Stream(dev)
            s.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(s):
                for c, sc in layers:  # warm-up on the capture stream (its cached workspace)
                    layer(c, sc, which)
            torch.cuda.current_stream(dev).wait_stream(s)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            reps = 4
            with torch.cuda.graph(g, stream=s):
                for _ in range(reps):
                    for c, sc in layers:
                        layer(c, sc, which)
            g.replay()
            torch.cuda.synchronize()
            ts = []
            for _ in range(replays):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda._sleep(300_000)
                a.record()
                g.replay()
                b.record()
                b.synchronize()
                ts.append(a.elapsed_time(b) * 1e3 / (reps * len(layers)))
            del g
            return float(np.median(ts))

        t_layer = graph_us()
        per = {nm: round(graph_us(nm), 2) for nm, _, _ in LAYER}
        by = decode_layer_bytes(m)
        gemm_floor_us = sum(n * k + m * k + 4.0 * (m * k / 128 + n * k / 16384) + 2.0 * m * n
                            for _, n, k in LAYER) / (peaks["hbm_gbs"] * 1e3)
        gbs = by / (t_layer * 1e-6) / 1e9
        out[f"m{m}"] = {"layer_us": round(t_layer, 2), "per_gemm_us_incl_act_quant": per,
                        "algorithmic_bytes": int(by), "GBps": round(gbs, 1),
                        "frac_hbm": round(gbs / peaks["hbm_gbs"], 4),
                        "gemm_hbm_floor_us": round(gemm_floor_us, 2),
                        "layer_tflops": round(layer_flops(m) / (t_layer * 1e-6) / 1e12, 2)}
    del layers
    return {"config": "BASELINE.json configs[2]: Qwen3-8B decode-shaped GEMMs (M tokens, real N, K), bf16 out; "
                      "each linear = fp8_linear_dynamic (BF16 input quantized per token per 128 channels + "
                      "blockwise FP8 GEMM, two kernels chained by programmatic dependent launch)",
            "timing": f"one CUDA graph of {copies} layers x 4 replays (weights rotate over {copies} copies, "
                      f"{copies} x 193 MB > L2), median of {replays} replays; per_gemm = graphs of one linear "
                      "(incl. its activation quantization) alone",
            "roofline": {"bound": "hbm", "unit": "GB/s", "peak": peaks["hbm_gbs"],
                         "achieved_by_m": {k: v["GBps"] for k, v in out.items()},
                         "frac_by_m": {k: v["frac_hbm"] for k, v in out.items()}},
            "results": out, "clocks": clocks.summary(t_win, time.perf_counter())}


def bench_moe(device, peaks, clocks, flush, tokens=(1024, 8192), iters=10):
    """C4 (BASELINE.json configs[3]): Qwen3-30B-A3B experts, 128 experts, top-8: fc1 (gate_up,
    [128][1536, 2048]) and fc2 (down, [128][2048, 768]) grouped blockwise FP8 GEMMs on the rows
    routed to each expert (device int32 offsets), uniform and Zipf(1.2)-skewed routing; also the
    EP-8 shard (16 experts per rank, the tokens routed to them)."""
    from paper_2601_18150_b200 import fp8q
    gen = torch.Generator(device=device)
    gen.manual_seed(4242)
    experts = {}
    for name, (E, n, k) in synth.QWEN3_30B_EXPERTS.items():
        w = dev_bf16((E * n, k), gen, device, 0.02)
        wq, ws = fp8q.quantize_weight_blockwise(w)
        del w
        experts[name] = (wq.view(E, n, k), ws.view(E, n // 128, k // 128), n, k)
    peak = fp8_peak_tflops(peaks, sustained=False)
    res = {}
    t_win = time.perf_counter()
    cases = [(T, 0.0, 128) for T in tokens] + [(max(tokens), 1.2, 128), (max(tokens), 0.0, 16)]
    for T, skew, E_used in cases:
        sizes = synth.moe_group_sizes(T, seed=0, skew=skew)
        if E_used < 128:  # EP-8: rank 0 owns experts [0, 16) and the rows routed to them
            sizes = sizes[:E_used]
        off = torch.from_numpy(synth.offsets_from_sizes(sizes)).to(device)
        rows = int(sizes.sum())
        rec = {"rows": rows, "experts": E_used, "rows_per_expert_min_max": [int(sizes.min()), int(sizes.max())]}
        for name, (wq, ws, n, k) in experts.items():
            x = dev_bf16((rows, k), gen, device)
            xq, xs = fp8q.quantize_act_per_token_group(x)
            y = torch.empty((rows, n), dtype=torch.bfloat16, device=device)
            wqe, wse = wq[:E_used], ws[:E_used]
            t = time_launch(lambda: fp8q.fp8_block_gemm_grouped(xq, xs, wqe, wse, off, out=y), flush, iters)
            flops = 2.0 * rows * n * k
            by = E_used * n * k + rows * k + 4.0 * (rows * k / 128 + E_used * n * k / 16384) + 2.0 * rows * n
            t_tc = flops / (peak * 1e12)
            t_hbm = by / (peaks["hbm_gbs"] * 1e9)
            rec[name] = {"shape_rows_n_k": [rows, n, k], "us": round(t * 1e3, 2),
                         "tflops_real_rows": round(flops / (t * 1e-3) / 1e12, 1),
                         "GBps": round(by / (t * 1e-3) / 1e9, 1),
                         "bound": "tensor" if t_tc > t_hbm else "hbm",
                         "frac_max_roofline": round(max(t_tc, t_hbm) / (t * 1e-3), 4)}
            del x, xq, xs, y
        key = f"T{T}_{'zipf1.2' if skew else 'uniform'}" + ("_ep8_16experts" if E_used < 128 else "")
        res[key] = rec
    del experts
    return {"config": "BASELINE.json configs[3]: Qwen3-30B-A3B experts (128 x fc1 [1536,2048], fc2 [2048,768]), "
                      "top-8 routing, bf16 out",
            "timing": f"CUDA events per launch after a 256 MB L2 flush (write + read back: cold, clean L2), median of {iters}",
            "roofline": {"bound": "max(tensor, hbm) per case", "tensor_peak_tflops": round(peak, 1),
                         "hbm_peak_gbs": peaks["hbm_gbs"],
                         "note": "tensor peak = 2 x measured bf16 BURST (kernels timed alone)"},
            "results": res, "clocks": clocks.summary(t_win, time.perf_counter())}


def model_specs(workload):
    """Every quantized linear weight of the model (Appendix C)."""
    from paper_2601_18150_b200.sync import TensorSpec
    specs = []
    if workload == "sync30b":
        for layer in range(synth.QWEN3_30B_LAYERS):
            for name, (n, k) in synth.QWEN3_30B_ATTN.items():
                specs.append(TensorSpec(f"L{layer}.{name}", n, k))
            for name, (e, n, k) in synth.QWEN3_30B_EXPERTS.items():
                specs.append(TensorSpec(f"L{layer}.experts.{name}", n, k, experts=e))
    else:
        for layer in range(synth.QWEN3_8B_LAYERS):
            for name, (n, k) in synth.QWEN3_8B_LINEARS.items():
                specs.append(TensorSpec(f"L{layer}.{name}", n, k))
    return specs


def bench_sync(workload, device, world, rank, peaks, clocks, steps=10, warmup=3, fanout=False):
    """C5 (BASELINE.json configs[4]): whole-model per-step weight sync -- each rank
    requantizes its 1/P of every weight (batched launches) and the FP8 codes/scales are
    all-gathered (grouped NCCL calls on a comm stream, overlapped) or, with fanout, stored by the
    quantizer straight into every rank's symmetric-memory buffer.  Strong scaling (fixed model)."""
    from paper_2601_18150_b200 import fp8q
    from paper_2601_18150_b200.sync import WeightSyncEngine, symmetric_peer_buffers
    specs = model_specs(workload)
    mode = "quantize shard + grouped NCCL all-gather" if world > 1 else "quantize (P = 1, no exchange)"
    peers = None
    if fanout and world > 1:
        try:
            peers = symmetric_peer_buffers(specs, device)
            mode = "fan-out quantizer (P2P stores into every rank's symmetric-memory buffer)"
        except Exception as exc:  # noqa: BLE001 - reported in the JSON line
            mode = f"gather (fan-out unavailable: {type(exc).__name__}: {exc})"[:200]
    eng = WeightSyncEngine(specs, device, peers=peers)
    gen = torch.Generator(device=device)
    shards = {}
    local_elems = 0
    for i, sp in enumerate(specs):
        r0, r1 = eng.shard_rows(sp.name)
        gen.manual_seed(1000 + i)
        shards[sp.name] = dev_bf16((r1 - r0, sp.k), gen, device, 0.02)
        local_elems += (r1 - r0) * sp.k
    total_elems = sum(sp.rows * sp.k for sp in specs)
    fp8_bytes = sum(sp.rows * sp.k + sp.scale_rows * sp.scale_cols * 4 for sp in specs)
    comm = torch.cuda.Stream(device) if world > 1 else None
    step = 0
    for _ in range(warmup):
        step += 1
        eng.sync_step(step, shards, comm, strict=False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_win = time.perf_counter()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    torch.cuda._sleep(2_000_000)
    for i in range(steps):
        step += 1
        evs[i][0].record()
        eng.sync_step(step, shards, comm, strict=False)
        evs[i][1].record()
    torch.cuda.synchronize()
    eng.check_finite()
    if world > 1:
        dist.barrier()
    ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in evs) / steps, device, world)
    algo_bytes = total_elems * WEIGHT_BYTES_PER_ELEM
    gbs = algo_bytes / (ms * 1e-3) / 1e9
    floor_q = algo_bytes / world / (peaks["hbm_gbs"] * 1e9) * 1e3
    floor_g = (world - 1) / world * fp8_bytes / 900e9 * 1e3 if world > 1 else 0.0
    rec = {"workload": f"{workload}_whole_model_weight_sync", "n_ranks": world, "tensors": len(specs),
           "quantized_params": total_elems, "fp8_bytes": fp8_bytes, "exchange": mode,
           "ms_per_sync": round(ms, 4), "aggregate_requant_GBps": round(gbs, 1),
           "per_rank_requant_GBps": round(local_elems * WEIGHT_BYTES_PER_ELEM / (ms * 1e-3) / 1e9, 1),
           "floor_quantize_ms": round(floor_q, 3), "floor_allgather_ms_900GBps": round(floor_g, 3),
           "frac_of_floor": round(max(floor_q, floor_g) / ms, 4),
           "roofline": {"bound": "hbm" if world == 1 else "max(hbm/P, nvlink ingress)",
                        "achieved": round(gbs, 1), "peak": peaks["hbm_gbs"] * world, "unit": "GB/s",
                        "frac": round(max(floor_q, floor_g) / ms, 4),
                        "kernel": "quantize_weight_blockwise_batched (TMA-staged, 16 tensors per launch)"},
           "clocks": clocks.summary(t_win, time.perf_counter()) if clocks else None}
    del eng, shards, peers
    torch.cuda.empty_cache()
    return rec


TP_SHAPES = {"qwen3_8b": [("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 24576, 4096), ("down", 4096, 12288)],
             "qwen3_30b_a3b_attn": [("qkv", 5120, 2048), ("o", 2048, 4096)]}


def bench_tp_shards(st: LayerStep, peaks, clocks, flush, ps=(2, 4, 8), iters=10):
    """north_star: "The GEMM is reported per GPU and as column-parallel shards":
    each rank multiplies the replicated M = 8192 activations by its N/P rows of W (and the
    matching scale rows); no collective inside the GEMM.  Per shard GEMM: per-GPU TFLOP/s and
    the fraction of the burst FP8 peak; aggregate = P x per-GPU (every rank runs its shard)."""
    from paper_2601_18150_b200 import fp8q
    dev = st.device
    m = st.m
    gen = torch.Generator(device=dev)
    gen.manual_seed(99)
    weights = {"qwen3_8b": {nm: (st.engine.codes[nm], st.engine.scales[nm]) for nm, _, _ in LAYER}}
    w30 = {}
    for nm, n, k in TP_SHAPES["qwen3_30b_a3b_attn"]:
        w30[nm] = fp8q.quantize_weight_blockwise(dev_bf16((n, k), gen, dev, 0.02))
    weights["qwen3_30b_a3b_attn"] = w30
    acts = {k: (st.xq[nm], st.xs[nm]) for nm, _, k in LAYER}
    x2048 = dev_bf16((m, 2048), gen, dev)
    acts[2048] = fp8q.quantize_act_per_token_group(x2048)
    peak = fp8_peak_tflops(peaks, sustained=False)
    res = {}
    t_win = time.perf_counter()
    for model, shapes in TP_SHAPES.items():
        for P in ps:
            rec, tot_f, tot_t = {}, 0.0, 0.0
            for nm, n, k in shapes:
                ns = n // P
                c, s = weights[model][nm]
                cs, ss = c[:ns], s[:(ns + 127) // 128]
                xq, xs = acts[k]
                y = torch.empty((m, ns), dtype=torch.bfloat16, device=dev)
                t = time_launch(lambda: fp8q.fp8_block_gemm(xq, xs, cs, ss, out=y), flush, iters)
                f = 2.0 * m * ns * k
                tot_f += f
                tot_t += t
                tf = f / (t * 1e-3) / 1e12
                rec[nm] = {"shape_m_n_k": [m, ns, k], "us": round(t * 1e3, 1), "tflops_per_gpu": round(tf, 1),
                           "frac_fp8_burst": round(tf / peak, 4)}
            per_gpu = tot_f / (tot_t * 1e-3) / 1e12
            rec["layer"] = {"tflops_per_gpu": round(per_gpu, 1), "tflops_aggregate": round(P * per_gpu, 1),
                            "frac_fp8_burst": round(per_gpu / peak, 4)}
            res[f"{model}_P{P}"] = rec
    del weights, w30, x2048
    return {"config": "column-parallel shard GEMMs (N/P rows of each weight, replicated M = 8192 activations)",
            "timing": f"CUDA events per launch after a 256 MB L2 flush (write + read back: cold, clean L2), median of {iters}",
            "roofline": {"bound": "tensor", "peak": round(peak, 1), "unit": "TFLOP/s",
                         "peak_source": "2 x measured bf16 BURST (kernels timed alone)"},
            "results": res, "clocks": clocks.summary(t_win, time.perf_counter())}


# ----------------------------------------------------------------------------- CPU oracle
_ORACLE_W = []
_ORACLE_X = {}


def oracle_inputs(rows):
    """Seeded host inputs for the oracle sample (generated once per process): the layer's four
    full BF16 weights and `rows` token rows of each activation."""
    if not _ORACLE_W:
        _ORACLE_W.extend(synth.qwen3_weight(n, k, seed=i) for i, (_, n, k) in enumerate(LAYER))
    if rows not in _ORACLE_X:
        _ORACLE_X[rows] = [synth.qwen3_activation(rows, k, seed=i) for i, (_, _, k) in enumerate(LAYER)]
    return list(zip(_ORACLE_W, _ORACLE_X[rows]))


def cpu_oracle_sample(rows, nth, requant=True):
    """The oracle as it stands on `nth` host threads: blockwise requant of the layer's four
    weights (full), per-token-group quantization of `rows` token rows of each input, and the
    fp64 GEMM of those rows against the full weights.  Returns (t_requant, t_act, t_gemm) s."""
    import oracle
    t_w = t_a = t_g = 0.0
    for wb, xb in oracle_inputs(rows):
        t0 = time.perf_counter()
        bq, bs = oracle.quantize_weight_blockwise(wb, nthreads=nth) if requant else (None, None)
        t1 = time.perf_counter()
        aq, as_ = oracle.quantize_act_per_token_group(xb, nthreads=nth)
        t2 = time.perf_counter()
        if bq is None:
            bq, bs = _cached_weight_codes(wb)
        oracle.gemm_rows(aq, as_, bq, bs, nthreads=nth)
        t3 = time.perf_counter()
        t_w += t1 - t0
        t_a += t2 - t1
        t_g += t3 - t2
    return t_w, t_a, t_g


_WCODES = {}


def _cached_weight_codes(wb):
    import oracle
    key = id(wb)
    if key not in _WCODES:
        _WCODES[key] = oracle.quantize_weight_blockwise(wb)
    return _WCODES[key]


def cpu_extrapolate(t_w, t_a, t_g, rows, m=M_PREFILL):
    """Full-step seconds: the whole requant + activation quant and GEMM scaled from `rows` to m."""
    return t_w + (t_a + t_g) * (m / rows)


def cpu_baseline_record(rows_all=8, rows_one=1):
    """BASELINE.md §4 CPU plan: the oracle at all host cores and at one thread, lscpu model,
    requant / activation-quant GB/s and fp64 GEMM GFLOP/s, extrapolated full-step time."""
    import oracle
    oracle.build()
    nth = oracle.default_threads()
    w_elems = sum(n * k for _, n, k in LAYER)
    gemm_flops_row = sum(2.0 * n * k for _, n, k in LAYER)
    act_elems_row = sum(k for _, _, k in LAYER)
    t0 = time.perf_counter()
    tw, ta, tg = cpu_oracle_sample(rows_all, nth)
    t_all = time.perf_counter() - t0
    full_all = cpu_extrapolate(tw, ta, tg, rows_all)
    t1 = time.perf_counter()
    tw1, ta1, tg1 = cpu_oracle_sample(rows_one, 1, requant=False)
    # one-thread requant on one weight (o_proj, 16.8 M elements), scaled to the layer
    import oracle as _o
    wb_o = oracle_inputs(rows_one)[1][0]
    tq0 = time.perf_counter()
    _o.quantize_weight_blockwise(wb_o, nthreads=1)
    tq1 = time.perf_counter() - tq0
    tw1 = tq1 * w_elems / wb_o.size
    t_one = time.perf_counter() - t1
    full_one = cpu_extrapolate(tw1, ta1, tg1, rows_one)
    val = layer_flops(M_PREFILL) / full_all / 1e12
    return {"value": round(val, 8), "unit": "TFLOP/s", "cores": nth, "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": f"all {nth} threads: full requant of the 4 layer weights ({w_elems / 1e6:.0f} M elements, "
                      f"{tw:.2f} s) + act quant ({ta:.2f} s) and fp64 GEMM ({tg:.2f} s) of {rows_all}/{M_PREFILL} "
                      f"token rows, extrapolated to one full step = {full_all:.1f} s",
            "measured_s": round(t_all, 2),
            "all_cores": {"threads": nth, "requant_GBps": round(w_elems * WEIGHT_BYTES_PER_ELEM / tw / 1e9, 3),
                          "act_quant_GBps": round(rows_all * act_elems_row * ACT_BYTES_PER_ELEM / ta / 1e9, 3),
                          "gemm_GFLOPs": round(rows_all * gemm_flops_row / tg / 1e9, 3),
                          "full_step_s_extrapolated": round(full_all, 1),
                          "whole_model_requant_s_extrapolated": {
                              "qwen3_8b": round(6.946e9 * WEIGHT_BYTES_PER_ELEM / (w_elems * WEIGHT_BYTES_PER_ELEM / tw), 1),
                              "qwen3_30b_a3b": round(29.897e9 * WEIGHT_BYTES_PER_ELEM / (w_elems * WEIGHT_BYTES_PER_ELEM / tw), 1)}},
            "one_thread": {"threads": 1, "requant_GBps": round(w_elems * WEIGHT_BYTES_PER_ELEM / tw1 / 1e9, 3),
                           "act_quant_GBps": round(rows_one * act_elems_row * ACT_BYTES_PER_ELEM / ta1 / 1e9, 3),
                           "gemm_GFLOPs": round(rows_one * gemm_flops_row / tg1 / 1e9, 3),
                           "full_step_s_extrapolated": round(full_one, 1), "measured_s": round(t_one, 2)}}


# ----------------------------------------------------------------------------- arms
def run_reference(args):
    """The reference arm of this tier: the CPU oracle, as it stands, on the host cores.  One
    step = the bounded sample (full requant of the layer's weights + activation quant and fp64
    GEMM of `rows` token rows); ms_per_step is that MEASURED sample time, value the throughput
    extrapolated to the full M = 8192 step (both stated)."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    nth = oracle.default_threads()
    rows = 2
    for _ in range(args.warmup):
        cpu_oracle_sample(rows, nth)
    tw = ta = tg = 0.0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        a, b, c = cpu_oracle_sample(rows, nth)
        tw += a
        ta += b
        tg += c
    measured = (time.perf_counter() - t0) / args.steps
    full_s = cpu_extrapolate(tw / args.steps, ta / args.steps, tg / args.steps, rows)
    val = layer_flops(M_PREFILL) / full_s / 1e12
    sample = (f"per step: full blockwise requant of the 4 Qwen3-8B layer weights (193M elements) + activation "
              f"quant and fp64 GEMM of {rows} of {M_PREFILL} token rows on {nth} threads; value extrapolated to "
              f"M={M_PREFILL} ({full_s:.1f} s per full step)")
    line = {"impl": "reference", "metric": METRIC, "value": round(val, 8), "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(measured * 1e3, 3),
            "extrapolated_ms_per_full_step": round(full_s * 1e3, 1),
            "value_basis": "layer GEMM FLOPs at M=8192 / extrapolated full-step time (ms_per_step = measured sample)",
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Qwen3-8B-shaped BF16 weights/activations)",
            "config": headline_config(world),
            "cpu_baseline": {"value": round(val, 8), "unit": "TFLOP/s", "cores": nth, "kind": "oracle",
                             "cpu_model": cpu_model(), "sample": sample},
            "e2e": {"value": round(val, 8), "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_layer(args):
    world, rank, local = dist_env()
    device = init_dist(world, local)
    peaks = load_peaks()
    from paper_2601_18150_b200 import fp8q
    fp8q.load_library()
    st = LayerStep(world, rank, device)
    clocks = ClockSampler(device.index)
    clocks.start()
    # >= W warm-up steps, and at least ~1.5 s of them so nvidia-smi sees the GPU under load
    t0 = time.perf_counter()
    done = 0
    while done < args.warmup or time.perf_counter() - t0 < 1.5:
        st.run()
        done += 1
        if done % 16 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = fp8q.kernel_launches()
    t_win0 = time.perf_counter()
    torch.cuda._sleep(2_000_000)  # GPU busy (~1 ms) while the host enqueues: no idle gap timed
    for i in range(args.steps):
        evs[i][0].record()
        st.run(evs[i])
        evs[i][3].record()
    torch.cuda.synchronize()
    t_win1 = time.perf_counter()
    launches = fp8q.kernel_launches() - launches0
    st.engine.check_finite()
    if world > 1:
        dist.barrier()
    t_step = [evs[i][0].elapsed_time(evs[i][3]) for i in range(args.steps)]
    t_sync = [evs[i][0].elapsed_time(evs[i][1]) for i in range(args.steps)]
    t_act = [evs[i][1].elapsed_time(evs[i][2]) for i in range(args.steps)]
    t_gemm = [evs[i][2].elapsed_time(evs[i][3]) for i in range(args.steps)]
    ms_per_step = max_over_ranks(sum(t_step), device, world) / args.steps

    flops_rank = layer_flops(st.m)
    value = flops_rank * world / (ms_per_step * 1e-3) / 1e12
    gemm_ms = float(np.mean(t_gemm))
    gemm_tflops = flops_rank / (gemm_ms * 1e-3) / 1e12
    peak = fp8_peak_tflops(peaks, sustained=True)
    peak_burst = fp8_peak_tflops(peaks, sustained=False)
    sync_ms = float(np.mean(t_sync))
    act_ms = float(np.mean(t_act))
    requant_gbs = st.weight_elems_local * WEIGHT_BYTES_PER_ELEM / (sync_ms * 1e-3) / 1e9
    act_gbs = st.act_elems * ACT_BYTES_PER_ELEM / (act_ms * 1e-3) / 1e9
    clk = clocks.summary(t_win0 - 1.5, t_win1)

    # e2e through the same C-ABI calls with host (pinned) buffers
    e2e_ms = None
    if not args.no_e2e:
        for _ in range(2):
            st.run_e2e()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2_000_000)
        e0.record()
        for _ in range(args.steps):
            st.run_e2e()
        e1.record()
        torch.cuda.synchronize()
        st.engine.check_finite()
        e2e_ms = max_over_ranks(e0.elapsed_time(e1), device, world) / args.steps

    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("fp8_block_gemm_bytes_per_launch")
        except Exception:
            traffic = None

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp8_e4m3 (fp32 accumulate)",
        "data": "synthetic (seeded Qwen3-8B-shaped BF16 weights/activations)",
        "config": headline_config(world, st.m),
        "breakdown": {"sync_ms": round(sync_ms, 4), "requant_gbs_local": round(requant_gbs, 1),
                      "requant_frac_hbm": round(requant_gbs / peaks["hbm_gbs"], 4) if world == 1 else None,
                      "act_quant_ms": round(act_ms, 4), "act_quant_gbs": round(act_gbs, 1),
                      "act_quant_frac_hbm": round(act_gbs / peaks["hbm_gbs"], 4),
                      "gemm_ms": round(gemm_ms, 4), "gemm_tflops": round(gemm_tflops, 1),
                      "gemm_frac_fp8_peak_sustained": round(gemm_tflops / peak, 4),
                      "gemm_frac_fp8_peak_burst": round(gemm_tflops / peak_burst, 4)},
        "roofline": {"bound": "tensor", "achieved": round(gemm_tflops, 1), "peak": round(peak, 1), "unit": "TFLOP/s",
                     "frac": round(gemm_tflops / peak, 4), "traffic": traffic,
                     "kernel": "fp8_block_gemm (4 launches/step; achieved = algorithmic GEMM FLOPs / CUDA-event time)",
                     "peak_source": "2 x bf16 SUSTAINED of " + peaks["source"] + " (steady-state, power-capped timing)"},
        "gpu_launches": int(launches),
        "warmup_steps_run": done,
        "clocks": clk,
        "paper_context": PAPER_CONTEXT,
    }
    if e2e_ms is not None:
        line["e2e"] = {"value": round(flops_rank * world / (e2e_ms * 1e-3) / 1e12, 3), "unit": "TFLOP/s",
                       "h2d_bytes_per_step": int(st.h2d_bytes()), "d2h_bytes_per_step": int(st.d2h_bytes()),
                       "ms_per_step": round(e2e_ms, 3)}

    # ---- the other §8(d) rows (rank 0 measures the single-GPU kernels; every rank the sync)
    if not args.no_extras:
        flush = L2Flush(device)
        if rank == 0:
            line["decode"] = bench_decode(st, peaks, clocks)
            line["tp_shards"] = bench_tp_shards(st, peaks, clocks, flush)
        del st
        torch.cuda.empty_cache()
        if rank == 0:
            line["moe"] = bench_moe(device, peaks, clocks, flush)
        torch.cuda.empty_cache()
        if world > 1:
            dist.barrier()
        line["sync"] = {w: bench_sync(w, device, world, rank, peaks, clocks) for w in ("sync8b", "sync30b")}
        del flush
    clocks.stop()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_record()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_single(args):
    """Development entry: one sub-record as its own JSON line (--workload decode|moe|shards|sync8b|sync30b)."""
    world, rank, local = dist_env()
    device = init_dist(world, local)
    peaks = load_peaks()
    clocks = ClockSampler(device.index)
    clocks.start()
    flush = L2Flush(device)
    if args.workload.startswith("sync"):
        rec = bench_sync(args.workload, device, world, rank, peaks, clocks, steps=args.steps,
                         warmup=args.warmup, fanout=args.fanout)
    elif args.workload == "moe":
        rec = bench_moe(device, peaks, clocks, flush)
    else:
        st = LayerStep(world, rank, device)
        st.run()
        torch.cuda.synchronize()
        rec = bench_decode(st, peaks, clocks) if args.workload == "decode" else bench_tp_shards(st, peaks, clocks, flush)
    clocks.stop()
    if rank == 0:
        print(json.dumps({"metric": METRIC, "workload": args.workload, "n_gpus": world, "record": rec}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def relaunch_under_torchrun(args, argv) -> int:
    """--gpus N > 1 without a torchrun environment: start N ranks on this node (one process per
    GPU, 127.0.0.1 rendezvous) running this same command line, NCCL_DEBUG=INFO."""
    if torch.cuda.device_count() < args.gpus:
        print(f"bench.py: --gpus {args.gpus} but only {torch.cuda.device_count()} CUDA device(s) visible",
              file=sys.stderr)
        return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *argv]
    return subprocess.call(cmd, env=env)


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["layer8b", "decode", "moe", "shards", "sync8b", "sync30b"],
                    default="layer8b")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="headline step only (no decode/moe/sync/shard records)")
    ap.add_argument("--fanout", action="store_true", help="sync workloads: NEXT-1 fan-out quantizer (N > 1)")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    world, _, _ = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        if args.impl == "reference":
            return run_reference(args)  # the CPU arm runs on rank 0 alone anyway
        return relaunch_under_torchrun(args, argv)
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args)
    if args.workload != "layer8b":
        return run_single(args)
    return run_layer(args)


if __name__ == "__main__":
    sys.exit(main())
