#!/usr/bin/env python3
"""Per-kernel timing sweep (CUDA events on the launching stream, L2 flushed between
iterations, median of N) for the three libfp8q kernels on the BASELINE.json shapes.
Development tool: bench.py is the contract; this prints one JSON line per case."""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2601_18150_b200 import fp8q  # noqa: E402

PEAKS = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}
HBM = PEAKS["hbm_gbs"]
FP8 = 2 * PEAKS["bf16_tflops"]


FLUSH_MODE = "write"


def do_flush(flush):
    if FLUSH_MODE == "write":
        flush.zero_()  # dirty lines: the next kernel also pays their write-back
    elif FLUSH_MODE == "read":
        flush.view(torch.int64).sum()  # clean eviction: L2 left holding read-only lines


def timeit(fn, iters, flush):
    ts = []
    for _ in range(3):
        fn()
    for _ in range(iters):
        do_flush(flush)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # keep the GPU busy while the host enqueues: otherwise the start event fires on an idle
        # GPU and the timing includes the binding's launch overhead (tens of microseconds)
        torch.cuda._sleep(400_000)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)), float(np.percentile(ts, 10)), float(np.percentile(ts, 90))


def graph_time(fn, w, min_bytes=400 << 20):
    """Steady-state time per launch: a CUDA graph of back-to-back launches, each on its own
    copy of the weights (copies together > L2, so every launch streams from HBM)."""
    nbytes = w.numel() * w.element_size()
    copies = [w] + [w.clone() for _ in range(min(64, max(1, -(-min_bytes // nbytes))) - 1)]
    launches = 4 * len(copies)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for c in copies:
            fn(c)  # warm-up on the capture stream (creates its cached workspace outside the graph)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(launches):
            fn(copies[i % len(copies)])
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(400_000)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) / launches)
    del g, copies
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--what", default="all")
    ap.add_argument("--decode", action="store_true")
    ap.add_argument("--moe", action="store_true")
    ap.add_argument("--flush", choices=["write", "read", "none"], default="write")
    ap.add_argument("--graph", action="store_true", help="decode: also time back-to-back launches in a CUDA graph")
    args = ap.parse_args()
    global FLUSH_MODE
    FLUSH_MODE = args.flush
    dev = torch.device("cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    M = 8192
    for name, (n, k) in synth.QWEN3_8B_LINEARS.items():
        w = (torch.randn((n, k), generator=g, device=dev) * 0.02).to(torch.bfloat16)
        x = torch.randn((M, k), generator=g, device=dev).to(torch.bfloat16)
        wq, ws = fp8q.quantize_weight_blockwise(w)
        xq, xs = fp8q.quantize_act_per_token_group(x)
        y = torch.empty((M, n), dtype=torch.bfloat16, device=dev)
        if args.what in ("all", "wq"):
            t, lo, hi = timeit(lambda: fp8q.quantize_weight_blockwise(w, wq, ws), args.iters, flush)
            gbs = n * k * (3 + 4 / 16384) / (t * 1e-3) / 1e9
            print(json.dumps({"kernel": "quantize_weight_blockwise", "shape": [n, k], "ms": round(t, 4),
                              "p10": round(lo, 4), "p90": round(hi, 4), "GBps": round(gbs, 1), "frac_hbm": round(gbs / HBM, 4)}))
        if args.what in ("all", "aq"):
            t, lo, hi = timeit(lambda: fp8q.quantize_act_per_token_group(x, xq, xs), args.iters, flush)
            gbs = M * k * (3 + 4 / 128) / (t * 1e-3) / 1e9
            print(json.dumps({"kernel": "quantize_act_per_token_group", "shape": [M, k], "ms": round(t, 4),
                              "p10": round(lo, 4), "p90": round(hi, 4), "GBps": round(gbs, 1), "frac_hbm": round(gbs / HBM, 4)}))
        if args.what in ("aqref",):
            # reference point for an HBM-bound 2 B -> 1 B element map: torch's own cast kernel
            t, lo, hi = timeit(lambda: x.to(torch.float8_e4m3fn), args.iters, flush)
            gbs = M * k * 3 / (t * 1e-3) / 1e9
            print(json.dumps({"kernel": "torch_cast_bf16_to_e4m3", "shape": [M, k], "ms": round(t, 4),
                              "GBps": round(gbs, 1), "frac_hbm": round(gbs / HBM, 4)}))
        if args.what in ("all", "gemm"):
            t, lo, hi = timeit(lambda: fp8q.fp8_block_gemm(xq, xs, wq, ws, out=y), args.iters, flush)
            tf = 2 * M * n * k / (t * 1e-3) / 1e12
            print(json.dumps({"kernel": "fp8_block_gemm", "shape": [M, n, k], "ms": round(t, 4), "p10": round(lo, 4),
                              "p90": round(hi, 4), "TFLOPs": round(tf, 1), "frac_fp8": round(tf / FP8, 4)}))
        if args.decode:
            for m in (1, 8, 64, 128, 256):
                xd = xq[:m]
                sd = xs[:, :m].contiguous() if False else xs
                yd = torch.empty((m, n), dtype=torch.bfloat16, device=dev)
                t, lo, hi = timeit(lambda: fp8q.fp8_block_gemm(xd, sd, wq, ws, out=yd), args.iters, flush)
                by = n * k + m * k + 4 * (m * k / 128 + n * k / 16384) + 2 * m * n
                rec = {"kernel": "fp8_block_gemm_decode", "shape": [m, n, k], "ms": round(t, 4),
                       "GBps": round(by / (t * 1e-3) / 1e9, 1), "frac_hbm": round(by / (t * 1e-3) / 1e9 / HBM, 4)}
                if args.graph:
                    tg = graph_time(lambda w: fp8q.fp8_block_gemm(xd, sd, w, ws, out=yd), wq)
                    rec.update({"graph_ms": round(tg, 4), "graph_GBps": round(by / (tg * 1e-3) / 1e9, 1),
                                "graph_frac_hbm": round(by / (tg * 1e-3) / 1e9 / HBM, 4)})
                print(json.dumps(rec))
    if args.what in ("all", "fanout"):
        # NEXT-1: one Qwen3-8B layer's requant (4 weights, one launch) stored to R destinations
        from paper_2601_18150_b200.sync import TensorSpec, local_replica_buffers
        specs = [TensorSpec(nm, n, k) for nm, (n, k) in synth.QWEN3_8B_LINEARS.items()]
        ws = {sp.name: (torch.randn((sp.n, sp.k), generator=g, device=dev) * 0.02).to(torch.bfloat16)
              for sp in specs}
        elems = sum(sp.n * sp.k for sp in specs)
        for R in (1, 2, 4, 8):
            from paper_2601_18150_b200.sync import WeightSyncEngine
            eng = WeightSyncEngine(specs, dev, peers=local_replica_buffers(specs, dev, R))
            step = [0]

            def run():
                step[0] += 1
                eng.sync_step(step[0], ws)
            t, lo, hi = timeit(run, args.iters, flush)
            by = elems * (2 + R * (1 + 4 / 16384))
            print(json.dumps({"kernel": "quantize_weight_blockwise_fanout", "destinations": R, "elements": elems,
                              "ms": round(t, 4), "GBps": round(by / (t * 1e-3) / 1e9, 1),
                              "frac_hbm": round(by / (t * 1e-3) / 1e9 / HBM, 4)}))
            del eng
    if args.what in ("all", "mx"):
        # NEXT-4: MXFP8 quantizer (2 + 1 + 1/32 B per element) and block-scaled GEMM, Qwen3-8B M = 8192
        M = 8192
        for name, (n, k) in synth.QWEN3_8B_LINEARS.items():
            w = (torch.randn((n, k), generator=g, device=dev) * 0.02).to(torch.bfloat16)
            x = torch.randn((M, k), generator=g, device=dev).to(torch.bfloat16)
            wq, ws = fp8q.mx_quantize(w)
            xq, xs = fp8q.mx_quantize(x)
            t, lo, hi = timeit(lambda: fp8q.mx_quantize(x, xq, xs), args.iters, flush)
            by = M * k * (3 + 1 / 32)
            print(json.dumps({"kernel": "mx_quantize", "shape": [M, k], "ms": round(t, 4),
                              "GBps": round(by / (t * 1e-3) / 1e9, 1), "frac_hbm": round(by / (t * 1e-3) / 1e9 / HBM, 4)}))
            y = torch.empty((M, n), dtype=torch.bfloat16, device=dev)
            t, lo, hi = timeit(lambda: fp8q.fp8_mx_gemm(xq, xs, wq, ws, out=y), args.iters, flush)
            tf = 2 * M * n * k / (t * 1e-3) / 1e12
            print(json.dumps({"kernel": "fp8_mx_gemm", "name": name, "shape": [M, n, k], "ms": round(t, 4),
                              "p10": round(lo, 4), "p90": round(hi, 4), "TFLOPs": round(tf, 1),
                              "frac_fp8": round(tf / FP8, 4)}))
    if args.what in ("all", "kv"):
        # NEXT-3: calibration amax (2 B/elem) and append (3 B/elem) on Qwen3-8B K (8 heads x 128)
        cols = 8 * 128
        for T in (8192, 512, 64):
            x = torch.randn((T, cols), generator=g, device=dev).to(torch.bfloat16)
            amax = torch.zeros(1, dtype=torch.int32, device=dev)
            t, lo, hi = timeit(lambda: fp8q.kv_amax_update(x, amax), args.iters, flush)
            tg = graph_time(lambda xx: fp8q.kv_amax_update(xx, amax), x)
            print(json.dumps({"kernel": "kv_amax_update", "shape": [T, cols], "ms": round(t, 4),
                              "GBps": round(2 * T * cols / (t * 1e-3) / 1e9, 1), "graph_ms": round(tg, 4),
                              "graph_frac_hbm": round(2 * T * cols / (tg * 1e-3) / 1e9 / HBM, 4)}))
            scale = fp8q.kv_scale_from_amax(amax)
            cache = torch.empty((T + 64, cols), dtype=torch.uint8, device=dev)
            slots = torch.randperm(T + 64, device=dev)[:T].to(torch.int32)
            t, lo, hi = timeit(lambda: fp8q.kv_quantize_append(x, scale, cache, slots), args.iters, flush)
            tg = graph_time(lambda xx: fp8q.kv_quantize_append(xx, scale, cache, slots), x)
            print(json.dumps({"kernel": "kv_quantize_append", "shape": [T, cols], "ms": round(t, 4),
                              "GBps": round(3 * T * cols / (t * 1e-3) / 1e9, 1), "graph_ms": round(tg, 4),
                              "graph_frac_hbm": round(3 * T * cols / (tg * 1e-3) / 1e9 / HBM, 4)}))
    if args.what in ("all", "prod"):
        M = 8192
        for k in (4096, 2048):
            x = torch.randn((M, k), generator=g, device=dev).to(torch.bfloat16)
            gam = torch.ones(k, dtype=torch.bfloat16, device=dev)
            xq = torch.empty((M, k), dtype=torch.uint8, device=dev)
            xs = torch.empty((k // 128, fp8q.act_scales_ld(M)), dtype=torch.float32, device=dev)
            t, lo, hi = timeit(lambda: fp8q.rmsnorm_quantize_act_per_token_group(x, gam, 1e-6, xq, xs), args.iters, flush)
            gbs = M * k * (3 + 4 / 128) / (t * 1e-3) / 1e9
            print(json.dumps({"kernel": "rmsnorm_quantize", "shape": [M, k], "ms": round(t, 4), "GBps": round(gbs, 1),
                              "frac_hbm": round(gbs / HBM, 4)}))
        for inter in (12288, 768):
            gu = torch.randn((M, 2 * inter), generator=g, device=dev).to(torch.bfloat16)
            xq = torch.empty((M, inter), dtype=torch.uint8, device=dev)
            xs = torch.empty((inter // 128, fp8q.act_scales_ld(M)), dtype=torch.float32, device=dev)
            t, lo, hi = timeit(lambda: fp8q.silu_mul_quantize_act_per_token_group(gu, xq, xs), args.iters, flush)
            gbs = M * inter * (5 + 4 / 128) / (t * 1e-3) / 1e9
            print(json.dumps({"kernel": "silu_mul_quantize", "shape": [M, inter], "ms": round(t, 4), "GBps": round(gbs, 1),
                              "frac_hbm": round(gbs / HBM, 4)}))
    if args.moe:
        for T, skew in ((8192, 0.0), (8192, 1.2), (1024, 0.0)):
            sizes = synth.moe_group_sizes(T, seed=0, skew=skew)
            off = torch.from_numpy(synth.offsets_from_sizes(sizes)).to(dev)
            rows = int(sizes.sum())
            for name, (E, n, k) in synth.QWEN3_30B_EXPERTS.items():
                w = (torch.randn((E * n, k), generator=g, device=dev) * 0.02).to(torch.bfloat16)
                wq, ws = fp8q.quantize_weight_blockwise(w)
                wq = wq.view(E, n, k)
                ws = ws.view(E, n // 128, k // 128)
                x = torch.randn((rows, k), generator=g, device=dev).to(torch.bfloat16)
                xq, xs = fp8q.quantize_act_per_token_group(x)
                y = torch.empty((rows, n), dtype=torch.bfloat16, device=dev)
                t, lo, hi = timeit(lambda: fp8q.fp8_block_gemm_grouped(xq, xs, wq, ws, off, out=y), args.iters, flush)
                tf = 2 * rows * n * k / (t * 1e-3) / 1e12
                by = E * n * k + rows * k + 2 * rows * n
                print(json.dumps({"kernel": "fp8_block_gemm_grouped", "T": T, "skew": skew, "name": name,
                                  "shape": [rows, n, k, E], "ms": round(t, 4), "TFLOPs": round(tf, 1),
                                  "frac_fp8": round(tf / FP8, 4), "GBps": round(by / (t * 1e-3) / 1e9, 1)}))


if __name__ == "__main__":
    main()
