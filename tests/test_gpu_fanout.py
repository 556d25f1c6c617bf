"""GPU parity of the NEXT-1 fan-out weight quantizer: one launch
quantizes a rank's shards and stores every code / scale into every destination buffer
(peer-mapped memory in the multi-GPU engine; here several buffers of this GPU stand in for the
peers).  Every destination must hold exactly the oracle's bytes; the sync engine in fan-out
mode must leave the same bytes in every destination that the gather mode leaves."""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2601_18150_b200 import fp8q
from paper_2601_18150_b200.sync import TensorSpec, WeightSyncEngine, local_replica_buffers
from tests.helpers import to_dev_bf16

pytestmark = pytest.mark.gpu


def test_fanout_every_destination_bit_exact():
    shapes = [(384, 512), (256, 1024), (640, 256)]
    ws = [synth.qwen3_weight(n, k, 30 + i) for i, (n, k) in enumerate(shapes)]
    R = 3
    codes = [[torch.zeros((n, k), dtype=torch.uint8, device="cuda") for _ in range(R)] for n, k in shapes]
    scales = [[torch.zeros(((n + 127) // 128, (k + 127) // 128), dtype=torch.float32, device="cuda")
               for _ in range(R)] for n, k in shapes]
    # one delta per destination must serve every tensor: lay the replicas out as one flat buffer
    # per destination with identical per-tensor offsets
    c_tot = sum(n * k for n, k in shapes)
    s_tot = sum(((n + 127) // 128) * ((k + 127) // 128) for n, k in shapes)
    cflat = [torch.zeros(c_tot, dtype=torch.uint8, device="cuda") for _ in range(R)]
    sflat = [torch.zeros(s_tot, dtype=torch.float32, device="cuda") for _ in range(R)]
    items, co, so = [], 0, 0
    views = []
    for i, (n, k) in enumerate(shapes):
        nb = ((n + 127) // 128, (k + 127) // 128)
        cv = [c[co:co + n * k].view(n, k) for c in cflat]
        sv = [s[so:so + nb[0] * nb[1]].view(*nb) for s in sflat]
        items.append((to_dev_bf16(ws[i]), cv[0], sv[0]))
        views.append((cv, sv))
        co += n * k
        so += nb[0] * nb[1]
    fp8q.quantize_weight_blockwise_fanout(items, [c.data_ptr() - cflat[0].data_ptr() for c in cflat],
                                          [s.data_ptr() - sflat[0].data_ptr() for s in sflat])
    torch.cuda.synchronize()
    for i, (n, k) in enumerate(shapes):
        oc, os_ = oracle.quantize_weight_blockwise(ws[i])
        cv, sv = views[i]
        for d in range(R):
            assert np.array_equal(cv[d].cpu().numpy(), oc), (i, d)
            assert np.array_equal(sv[d].cpu().numpy().view(np.uint32), os_.view(np.uint32)), (i, d)


def test_fanout_validation():
    w = torch.zeros((128, 200), dtype=torch.bfloat16, device="cuda")  # k % 16 != 0: not wide
    c = torch.zeros((128, 200), dtype=torch.uint8, device="cuda")
    s = torch.zeros((1, 2), dtype=torch.float32, device="cuda")
    with pytest.raises(fp8q.Fp8qError, match="UNSUPPORTED"):
        fp8q.quantize_weight_blockwise_fanout([(w, c, s)], [0], [0])
    w2 = torch.zeros((128, 256), dtype=torch.bfloat16, device="cuda")
    c2 = torch.zeros((128, 256), dtype=torch.uint8, device="cuda")
    with pytest.raises(fp8q.Fp8qError, match="ALIGN"):
        fp8q.quantize_weight_blockwise_fanout([(w2, c2, s)], [0, 8], [0, 4])
    with pytest.raises(fp8q.Fp8qError, match="INVAL"):
        fp8q.quantize_weight_blockwise_fanout([(w2, c2, s)], [], [])


def test_engine_fanout_mode_matches_gather_mode():
    specs = [TensorSpec("qkv", 640, 512), TensorSpec("o", 512, 640), TensorSpec("experts", 256, 384, experts=3)]
    shards = {s.name: to_dev_bf16(synth.qwen3_weight(s.rows, s.k, 50 + i)) for i, s in enumerate(specs)}
    ref = WeightSyncEngine(specs, "cuda")
    ref.sync_step(1, shards)
    peers = local_replica_buffers(specs, "cuda", replicas=4)
    eng = WeightSyncEngine(specs, "cuda", peers=peers)
    eng.sync_step(1, shards)
    torch.cuda.synchronize()
    base_c, base_s = peers.codes_flat.data_ptr(), peers.scales_flat.data_ptr()
    reps_c, reps_s = peers._keep
    for s in specs:
        for d in range(4):
            # the engine's view of tensor s, re-based on destination d
            off_c = eng.codes[s.name].data_ptr() - base_c
            off_s = (eng.scales[s.name].data_ptr() - base_s) // 4
            got_c = reps_c[d][off_c:off_c + s.rows * s.k].view(s.rows, s.k)
            got_s = reps_s[d][off_s:off_s + s.scale_rows * s.scale_cols].view(s.scale_rows, s.scale_cols)
            assert torch.equal(got_c, ref.codes[s.name]), (s.name, d)
            assert torch.equal(got_s.view(torch.int32), ref.scales[s.name].view(torch.int32)), (s.name, d)
