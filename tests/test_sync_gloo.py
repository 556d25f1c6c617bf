"""Multi-process (gloo, CPU) tests of the sharded weight sync's host logic: shard planning,
in-place all-gather layout, step tags.  The quantizer is injected (the oracle), so the
gathered FP8 buffers on every rank must equal the oracle applied to the FULL weight,
bitwise (reading Q17), for world sizes 1 and 2 (and 4 via planning)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2601_18150_b200.sync import (StaleStepError, TensorSpec, WeightSyncEngine,
                                        plan_shards)

SPECS = [TensorSpec("qkv", 768, 256), TensorSpec("o", 256, 384),
         TensorSpec("experts_fc1", 256, 256, experts=4)]


def oracle_quantize(w: torch.Tensor, codes: torch.Tensor, scales: torch.Tensor) -> None:
    bits = w.view(torch.int16).numpy().view(np.uint16)
    c, s = oracle.quantize_weight_blockwise(np.ascontiguousarray(bits), nthreads=2)
    codes.copy_(torch.from_numpy(c))
    scales.copy_(torch.from_numpy(s))


def full_weight(spec: TensorSpec, step: int) -> torch.Tensor:
    bits = synth.qwen3_weight(spec.rows, spec.k, seed=1000 * step + len(spec.name))
    return torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        eng = WeightSyncEngine(SPECS, "cpu", quantize_fn=oracle_quantize)
        for step in (1, 2):
            shards = {}
            for s in SPECS:
                r0, r1 = eng.shard_rows(s.name)
                shards[s.name] = full_weight(s, step)[r0:r1].contiguous()
            eng.sync_step(step, shards)
            for s in SPECS:
                w = full_weight(s, step).view(torch.int16).numpy().view(np.uint16)
                oc, os_ = oracle.quantize_weight_blockwise(w, nthreads=2)
                assert np.array_equal(eng.codes[s.name].numpy(), oc), (rank, s.name)
                assert np.array_equal(eng.scales[s.name].numpy(), os_), (rank, s.name)
        try:
            eng.sync_step(2, shards)
            raise AssertionError("stale step accepted")
        except StaleStepError:
            pass
        assert eng.loaded_step == 2
        # buckets of one tensor with a completion hook (the e2e pipeline's mode): the hook sees
        # every tensor once, in spec order, after its gather; the bytes are unchanged
        seen = []
        shards = {}
        for s in SPECS:
            r0, r1 = eng.shard_rows(s.name)
            shards[s.name] = full_weight(s, 3)[r0:r1].contiguous()
        eng.sync_step(3, shards, bucket=1, on_bucket=seen.extend)
        assert seen == [s.name for s in SPECS], seen
        for s in SPECS:
            w = full_weight(s, 3).view(torch.int16).numpy().view(np.uint16)
            oc, os_ = oracle.quantize_weight_blockwise(w, nthreads=2)
            assert np.array_equal(eng.codes[s.name].numpy(), oc), (rank, s.name, "bucket=1")
            assert np.array_equal(eng.scales[s.name].numpy(), os_), (rank, s.name, "bucket=1")
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


@pytest.mark.parametrize("world", [1, 2])
def test_sharded_sync_equals_full_quantization(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in results.values()), results


def test_plan_shards_covers_and_aligns():
    for world in (1, 2, 4, 8):
        for spec in [TensorSpec("qkv", 6144, 4096), TensorSpec("gate_up", 24576, 4096),
                     TensorSpec("down", 4096, 12288), TensorSpec("e", 1536, 2048, experts=128),
                     TensorSpec("qkv30", 5120, 2048)]:
            plan = plan_shards(spec, world)
            assert plan[0].row0 == 0 and plan[-1].row1 == spec.rows
            assert plan[0].srow0 == 0 and plan[-1].srow1 == spec.scale_rows
            for a, b in zip(plan, plan[1:]):
                assert a.row1 == b.row0 and a.srow1 == b.srow0
            sizes = {p.row1 - p.row0 for p in plan}
            assert len(sizes) == 1 and all(p.row0 % 128 == 0 for p in plan)


def test_plan_rejects_indivisible():
    with pytest.raises(ValueError):
        plan_shards(TensorSpec("k30", 512, 2048), 8)  # 4 block-rows over 8 ranks (finding 10)
    with pytest.raises(ValueError):
        plan_shards(TensorSpec("e", 1536, 2048, experts=6), 4)
