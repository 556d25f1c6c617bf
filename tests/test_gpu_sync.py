"""GPU parity of the per-step weight sync: the
`WeightSyncEngine` on CUDA, through the C-ABI quantizers, must leave in its engine buffers
exactly the bytes of the ORACLE applied to the full BF16 weights -- for a whole Qwen3-8B layer
(qkv, o, gate_up, down at their real shapes) plus the real Qwen3-30B-A3B expert down projection
([128][2048, 768]) -- in every mode the bench and the e2e pipeline use:
  * gather mode, one batched launch per bucket of 16 tensors;
  * bucket = 1 with per-tensor `ready` events (uploads on another stream) and `on_bucket`;
  * NEXT-1 fan-out mode, every destination buffer.
Also: non-finite input is rejected (strict and deferred), a bad shard is rejected before
anything is launched, stale steps are rejected.  The world-2 NCCL test (gather + symmetric-
memory fan-out across two GPUs) runs where two GPUs are visible and is skipped otherwise."""
import os
import socket

import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2601_18150_b200.sync import (NonFiniteWeightError, StaleStepError, TensorSpec,
                                        WeightSyncEngine, local_replica_buffers)
from tests.helpers import to_dev_bf16

pytestmark = pytest.mark.gpu

SPECS = [TensorSpec(name, n, k) for name, (n, k) in synth.QWEN3_8B_LINEARS.items()]
SPECS.append(TensorSpec("experts.down", 2048, 768, experts=128))


@pytest.fixture(scope="module")
def model():
    """Full BF16 weights (host bits), their oracle bytes, and device copies."""
    host, ref, dev = {}, {}, {}
    for i, s in enumerate(SPECS):
        bits = synth.qwen3_weight(s.rows, s.k, seed=700 + i)
        host[s.name] = bits
        ref[s.name] = oracle.quantize_weight_blockwise(bits)
        dev[s.name] = to_dev_bf16(bits)
    return host, ref, dev


def _assert_engine_equals_oracle(codes, scales, ref, tag):
    for s in SPECS:
        oc, os_ = ref[s.name]
        assert torch.equal(codes[s.name], torch.from_numpy(oc).cuda()), (tag, s.name, "codes")
        got = scales[s.name].view(torch.int32)
        assert torch.equal(got, torch.from_numpy(os_.view(np.int32)).cuda()), (tag, s.name, "scales")


def test_sync_gather_mode_bit_exact(model):
    _, ref, dev = model
    eng = WeightSyncEngine(SPECS, "cuda")
    eng.sync_step(1, dev)
    torch.cuda.synchronize()
    _assert_engine_equals_oracle(eng.codes, eng.scales, ref, "gather")
    assert eng.loaded_step == 1 and not eng.poisoned
    with pytest.raises(StaleStepError):
        eng.sync_step(1, dev)


def test_sync_bucket1_ready_on_bucket_bit_exact(model):
    """The e2e pipeline's mode: shards uploaded on a side stream, each tensor quantized as soon
    as its upload event fires, a completion hook per tensor in spec order."""
    host, ref, _ = model
    eng = WeightSyncEngine(SPECS, "cuda")
    pinned = {s.name: torch.from_numpy(host[s.name].view(np.int16)).view(torch.bfloat16).pin_memory() for s in SPECS}
    shards = {s.name: torch.empty((s.rows, s.k), dtype=torch.bfloat16, device="cuda") for s in SPECS}
    up = torch.cuda.Stream()
    up.wait_stream(torch.cuda.current_stream())
    ready = {}
    with torch.cuda.stream(up):
        for s in SPECS:
            shards[s.name].copy_(pinned[s.name], non_blocking=True)
            ready[s.name] = torch.cuda.Event()
            ready[s.name].record(up)
    seen, done = [], {}

    def hook(names):
        for nm in names:
            seen.append(nm)
            done[nm] = torch.cuda.Event()
            done[nm].record(torch.cuda.current_stream())

    eng.sync_step(1, shards, bucket=1, ready=ready, on_bucket=hook)
    assert seen == [s.name for s in SPECS]
    for s in SPECS:
        done[s.name].synchronize()
    torch.cuda.synchronize()
    _assert_engine_equals_oracle(eng.codes, eng.scales, ref, "bucket=1")


def test_sync_fanout_mode_every_destination_bit_exact(model):
    _, ref, dev = model
    R = 2
    peers = local_replica_buffers(SPECS, "cuda", replicas=R)
    eng = WeightSyncEngine(SPECS, "cuda", peers=peers)
    eng.sync_step(1, dev)
    torch.cuda.synchronize()
    base_c, base_s = peers.codes_flat.data_ptr(), peers.scales_flat.data_ptr()
    reps_c, reps_s = peers._keep
    for d in range(R):
        codes, scales = {}, {}
        for s in SPECS:
            off_c = eng.codes[s.name].data_ptr() - base_c
            off_s = (eng.scales[s.name].data_ptr() - base_s) // 4
            codes[s.name] = reps_c[d][off_c:off_c + s.rows * s.k].view(s.rows, s.k)
            scales[s.name] = reps_s[d][off_s:off_s + s.scale_rows * s.scale_cols].view(s.scale_rows, s.scale_cols)
        _assert_engine_equals_oracle(codes, scales, ref, f"fanout dest {d}")


def test_sync_rejects_nonfinite_strict_and_deferred(model):
    _, ref, dev = model
    bad = dict(dev)
    w = dev["down"].clone()
    w[17, 4000] = float("nan")
    bad["down"] = w
    eng = WeightSyncEngine(SPECS, "cuda")
    eng.sync_step(1, dev)
    with pytest.raises(NonFiniteWeightError):
        eng.sync_step(2, bad)
    assert eng.loaded_step == 1 and eng.poisoned
    eng.sync_step(3, dev)  # a clean step restores the engine
    torch.cuda.synchronize()
    assert eng.loaded_step == 3 and not eng.poisoned
    _assert_engine_equals_oracle(eng.codes, eng.scales, ref, "after reject")
    # deferred: no host sync in sync_step; check_finite() reports it (and re-arms)
    inf = dict(dev)
    w2 = dev["experts.down"].clone()
    w2[-1, 0] = float("-inf")
    inf["experts.down"] = w2
    eng.sync_step(4, inf, strict=False)
    with pytest.raises(NonFiniteWeightError):
        eng.check_finite()
    eng.check_finite()  # flag re-armed
    # fan-out mode carries the flag too
    peers = local_replica_buffers(SPECS, "cuda", replicas=2)
    feng = WeightSyncEngine(SPECS, "cuda", peers=peers)
    with pytest.raises(NonFiniteWeightError):
        feng.sync_step(1, bad)
    assert feng.loaded_step == -1


def test_sync_validates_every_shard_before_launching(model):
    _, _, dev = model
    eng = WeightSyncEngine(SPECS, "cuda")
    for s in SPECS:
        eng.codes[s.name].fill_(0xA5)
    bad = dict(dev)
    bad["experts.down"] = dev["experts.down"][:-128]  # wrong shape, LAST tensor / bucket
    with pytest.raises(ValueError):
        eng.sync_step(1, bad, bucket=1)
    torch.cuda.synchronize()
    for s in SPECS:  # nothing was quantized: the first buckets did not run either
        assert bool((eng.codes[s.name] == 0xA5).all()), s.name
    bad["experts.down"] = dev["experts.down"].float()
    with pytest.raises(ValueError):
        eng.sync_step(1, bad)
    assert eng.loaded_step == -1


# ---------------------------------------------------------------------- world 2 (NCCL)
W2_SPECS = [TensorSpec("qkv", 6144, 4096), TensorSpec("o", 4096, 4096),
            TensorSpec("experts.down", 2048, 768, experts=16)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _w2_worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2601_18150_b200.sync import symmetric_peer_buffers
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(rank)
        dev = torch.device("cuda", rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
        full = {s.name: synth.qwen3_weight(s.rows, s.k, seed=900 + i) for i, s in enumerate(W2_SPECS)}
        ref = {n: oracle.quantize_weight_blockwise(b) for n, b in full.items()}
        modes = ["gather"]
        try:
            peers = symmetric_peer_buffers(W2_SPECS, dev)
            modes.append("fanout")
        except Exception as exc:  # noqa: BLE001 - reported, the test then fails
            q.put((rank, f"symmetric memory unavailable: {exc!r}"))
            return
        for mode in modes:
            eng = WeightSyncEngine(W2_SPECS, dev, peers=peers if mode == "fanout" else None)
            shards = {}
            for s in W2_SPECS:
                r0, r1 = eng.shard_rows(s.name)
                shards[s.name] = to_dev_bf16(full[s.name][r0:r1], dev)
            comm = torch.cuda.Stream(dev)
            eng.sync_step(1, shards, comm)
            torch.cuda.synchronize()
            for s in W2_SPECS:
                oc, os_ = ref[s.name]
                assert np.array_equal(eng.codes[s.name].cpu().numpy(), oc), (rank, mode, s.name)
                assert np.array_equal(eng.scales[s.name].cpu().numpy().view(np.uint32), os_.view(np.uint32)), \
                    (rank, mode, s.name)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs (NCCL world 2)")
def test_sync_world2_nccl_gather_and_fanout_bit_exact():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_w2_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in results.values()), results
