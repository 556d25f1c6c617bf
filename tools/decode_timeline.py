"""Dev: per-CTA launch timeline of one Qwen3-8B decode layer (4 x fp8_linear_dynamic) from the
trace build (`python paper_2601_18150_b200/build.py --trace` -> libfp8q_trace.so, -DFP8Q_TRACE).

Events (csrc/trace.cuh, globaltimer ns): GEMM 0 entry, 1 producer past griddepcontrol.wait,
2 last TMA issued, 3 first stage full (MMA), 4 last MMA issued, 5 promotion past the wait,
6 last k-block promoted, 7 exit; activation quantizer 10 entry, 11 past the wait, 12 exit.
Prints, per launch in start order, the min / median / max of every event relative to the
layer's first event (us).  Usage: python tools/decode_timeline.py [--m 1] [--copies 4]
"""
from __future__ import annotations

import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("FP8Q_LIB", os.path.join(ROOT, "paper_2601_18150_b200", "libfp8q_trace.so"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2601_18150_b200 import fp8q  # noqa: E402

NAMES = {0: "entry", 1: "p_wait", 2: "p_last", 3: "mma_1st", 4: "mma_last", 5: "e_wait", 6: "e_done",
         7: "exit", 10: "entry", 11: "wait", 12: "exit"}


def dump(lib, fn):
    cap = 1 << 20
    buf = np.zeros((cap, 4), dtype=np.uint32)
    n = ctypes.c_uint32(0)
    f = getattr(lib, fn)
    f.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint32)]
    if f(buf.ctypes.data, cap, ctypes.byref(n)) != 0:
        raise RuntimeError(fn)
    return buf[: n.value]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=1)
    ap.add_argument("--copies", type=int, default=4)
    args = ap.parse_args()
    lib = fp8q.load_library()
    dev = torch.device("cuda")
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    layer = [(nm,) + synth.QWEN3_8B_LINEARS[nm] for nm in ("qkv", "o", "gate_up", "down")]
    copies = []
    for _ in range(args.copies):
        c, s = {}, {}
        for nm, n, k in layer:
            mag = torch.randint(0, 0x7F, (n, k), generator=g, device=dev, dtype=torch.int32)
            sign = torch.randint(0, 2, (n, k), generator=g, device=dev, dtype=torch.int32) << 7
            c[nm] = (mag | sign).to(torch.uint8)
            s[nm] = torch.rand(((n + 127) // 128, k // 128), generator=g, device=dev) * 1e-3 + 1e-4
        copies.append((c, s))
    xs = {nm: torch.randn((args.m, k), generator=g, device=dev).to(torch.bfloat16) for nm, _, k in layer}
    ys = {nm: torch.empty((args.m, n), dtype=torch.bfloat16, device=dev) for nm, n, _ in layer}
    tags = {}
    for i, (c, s) in enumerate(copies):
        for nm, _, _ in layer:
            tags[s[nm].data_ptr() & 0xFFFFFFFF] = f"gemm {nm}#{i}"
    for nm, _, _ in layer:
        tags[xs[nm].data_ptr() & 0xFFFFFFFF] = f"aq {nm}"

    st = torch.cuda.Stream(dev)
    st.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(st):
        for c, s in copies:
            for nm, _, _ in layer:
                fp8q.fp8_linear_dynamic(xs[nm], c[nm], s[nm], out=ys[nm])
    torch.cuda.current_stream(dev).wait_stream(st)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=st):
        for c, s in copies:
            for nm, _, _ in layer:
                fp8q.fp8_linear_dynamic(xs[nm], c[nm], s[nm], out=ys[nm])
    graph.replay()
    torch.cuda.synchronize()
    dump(lib, "fp8q_trace_dump_skinny")
    dump(lib, "fp8q_trace_dump_quant")
    torch.cuda._sleep(200_000)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    graph.replay()
    b.record()
    torch.cuda.synchronize()
    total_us = a.elapsed_time(b) * 1e3
    rec = np.concatenate([dump(lib, "fp8q_trace_dump_skinny"), dump(lib, "fp8q_trace_dump_quant")])
    ap_out = os.environ.get("FP8Q_TIMELINE_NPZ")
    if ap_out:  # raw records + tag names for offline analysis
        np.savez(ap_out, rec=rec, tags=np.array(list(tags.keys()), dtype=np.uint32),
                 names=np.array(list(tags.values())))
    t = (rec[:, 2].astype(np.uint64) >> np.uint64(8) << np.uint64(32)) | rec[:, 3].astype(np.uint64)
    ev = rec[:, 2] & 0xFF
    t0 = t.min()
    rel = (t - t0).astype(np.float64) / 1e3
    launches = {}
    for tag in np.unique(rec[:, 0]):
        sel = rec[:, 0] == tag
        # a tag recurs once per graph pass only for the activation quantizer (same x every copy):
        # split its records into launches by entry order
        launches.setdefault(int(tag), []).append(sel)
    rows = []
    for tag, sels in launches.items():
        sel = sels[0]
        name = tags.get(tag, hex(tag))
        evs = ev[sel]
        rs = rel[sel]
        if name.startswith("aq"):
            # one CTA per launch at decode sizes: each entry/wait/exit triple is one launch
            order = np.argsort(rs)
            entries = sorted(rs[evs == 10])
            for i, e0 in enumerate(entries):
                e1 = entries[i + 1] if i + 1 < len(entries) else np.inf
                w = (rs >= e0) & (rs < e1)
                d = {NAMES[k]: rs[w & (evs == k)] for k in (10, 11, 12)}
                rows.append((e0, f"{name}[{i}]", d, ""))
            del order
        else:
            d = {NAMES[k]: rs[evs == k] for k in range(8)}
            # SM placement: CTAs sharing an SM with another CTA of the same launch, and when
            # their weight stream ended (event 2) against the others'
            sm = rec[sel, 1] >> 20
            cta = rec[sel, 1] & 0xFFFFF
            e0 = evs == 0
            sm_of = dict(zip(cta[e0].tolist(), sm[e0].tolist()))
            cnt = {}
            for v in sm_of.values():
                cnt[v] = cnt.get(v, 0) + 1
            doubled = {c for c, v in sm_of.items() if cnt[v] > 1}
            e2 = evs == 2
            pl = dict(zip(cta[e2].tolist(), rs[e2].tolist()))
            dbl = [pl[c] for c in doubled if c in pl]
            sgl = [v for c, v in pl.items() if c not in doubled]
            extra = (f"; SMs used {len(cnt)}, CTAs on shared SMs {len(doubled)}"
                     + (f" (p_last med {np.median(dbl):.1f} vs {np.median(sgl):.1f})" if dbl and sgl else ""))
            rows.append((rs.min(), name + f" ({int((evs == 0).sum())} CTAs)", d, extra))
    rows.sort(key=lambda r: r[0])
    print(f"M = {args.m}: graph of {len(copies)} layers, {total_us:.1f} us total "
          f"({total_us / len(copies):.1f} per layer); event times min/med/max us from the first event")
    for _, name, d, extra in rows:
        parts = []
        for k, v in d.items():
            if len(v):
                parts.append(f"{k} {v.min():.1f}/{np.median(v):.1f}/{v.max():.1f}")
        print(f"{name:24s} " + "  ".join(parts) + extra)


if __name__ == "__main__":
    main()
