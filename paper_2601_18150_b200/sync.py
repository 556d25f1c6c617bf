"""Sharded per-step weight synchronisation (§2.1.2, lines 67-75; SURVEY §8(a) a4,
§8(e)): "At each RL step, BF16/FP16 weights are retrieved from the training backend ...,
quantized to FP8 using the blockwise scheme ..., and loaded into the inference engine"
(PAPER.md:72).

B200 design: with P ranks (one process per GPU), rank r owns a contiguous
range of 128-row block-rows of every dense weight (or a contiguous range of experts of every
MoE weight), exactly the slice an FSDP-style sharded trainer holds.  Each rank quantizes
ONLY its slice, straight into its slot of the persistent full-size FP8 engine buffers, then
one in-place all-gather per buffer (NCCL over NVLink) fills the other slots.  Block-aligned
shards are independent, so the gathered bytes equal quantizing the full weight (reading Q17,
checked bitwise in the tests), and FP8 is gathered instead of BF16 (half the NVLink bytes).

Host logic here (planning, step tags, collectives) is plain Python over torch.distributed;
the quantizer is the libfp8q kernel.  `quantize_fn` is injectable only so the CPU gloo tests
can exercise the sharding and gather layout without a GPU.
"""
from __future__ import annotations

import dataclasses
from typing import Callable, Dict, List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist

BLOCK = 128


class StaleStepError(RuntimeError):
    """sync_step called with a step not newer than the loaded one."""


class NonFiniteWeightError(RuntimeError):
    """A shard held NaN/Inf (non-finite input is rejected).  The engine buffers are
    then undefined (`engine.poisoned`) and `loaded_step` is not advanced."""


@dataclasses.dataclass(frozen=True)
class TensorSpec:
    """One quantized linear weight.  Dense: [n, k] (nn.Linear [out, in]).  MoE experts:
    experts > 0 and the weight is [experts, n, k] (stored as [experts * n, k])."""
    name: str
    n: int
    k: int
    experts: int = 0

    @property
    def rows(self) -> int:
        return self.n * max(self.experts, 1)

    @property
    def scale_rows(self) -> int:
        return max(self.experts, 1) * ((self.n + BLOCK - 1) // BLOCK)

    @property
    def scale_cols(self) -> int:
        return (self.k + BLOCK - 1) // BLOCK


@dataclasses.dataclass(frozen=True)
class Shard:
    """Rows [row0, row1) of the (flattened) weight and scale rows [srow0, srow1) on one rank."""
    row0: int
    row1: int
    srow0: int
    srow1: int


def plan_shards(spec: TensorSpec, world: int) -> List[Shard]:
    """Split a weight into `world` equal, 128-row-block-aligned shards.

    Dense: rank r gets block-rows [r*B/P, (r+1)*B/P) with B = ceil(n/128) (requires B % P == 0
    so every rank's slot has the same size for the in-place all-gather; finding 10 of the
    survey: every Qwen3 fused tensor satisfies this for P <= 8).  MoE: rank r gets experts
    [r*E/P, (r+1)*E/P) (E % P == 0)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    if spec.experts:
        if spec.experts % world:
            raise ValueError(f"{spec.name}: {spec.experts} experts not divisible by {world} ranks")
        if spec.n % BLOCK:
            raise ValueError(f"{spec.name}: expert rows {spec.n} must be a multiple of {BLOCK}")
        per = spec.experts // world
        sb = spec.n // BLOCK
        return [Shard(r * per * spec.n, (r + 1) * per * spec.n, r * per * sb, (r + 1) * per * sb)
                for r in range(world)]
    nb = (spec.n + BLOCK - 1) // BLOCK
    if nb % world:
        raise ValueError(f"{spec.name}: {nb} block-rows not divisible by {world} ranks")
    if world > 1 and spec.n % BLOCK:
        raise ValueError(f"{spec.name}: sharded weights need n % {BLOCK} == 0")
    per = nb // world
    return [Shard(r * per * BLOCK, min((r + 1) * per * BLOCK, spec.n), r * per, (r + 1) * per)
            for r in range(world)]


QuantizeFn = Callable[[torch.Tensor, torch.Tensor, torch.Tensor], None]


class PeerBuffers:
    """NEXT-1: engine buffers of identical layout on several destinations.  The
    fan-out quantizer stores every code / scale of this rank's shard at pointer + delta[d] for
    each destination d, so every rank's engine buffer receives the shard straight from the
    quantizer (P2P stores over NVLink) and no all-gather pass re-reads it.

    codes_flat / scales_flat are this rank's (local) flat buffers; the engine lays its
    per-tensor views into them.  `fence()` orders the peers' later reads after the stores."""

    def __init__(self, codes_flat, scales_flat, codes_delta, scales_delta, fence=None, keep=()):
        self.codes_flat = codes_flat
        self.scales_flat = scales_flat
        self.codes_delta = [int(d) for d in codes_delta]
        self.scales_delta = [int(d) for d in scales_delta]
        self._fence = fence
        self._keep = keep  # owners of the destination memory

    def fence(self) -> None:
        if self._fence is not None:
            self._fence()


def _layout(specs):
    """Byte / element offsets of each tensor's codes and scales in the flat buffers (256-B aligned)."""
    co, so, c_off, s_off = {}, {}, 0, 0
    for s in specs:
        co[s.name] = c_off
        so[s.name] = s_off
        c_off += -(-(s.rows * s.k) // 256) * 256
        s_off += -(-(s.scale_rows * s.scale_cols) // 64) * 64
    return co, so, c_off, s_off


def local_replica_buffers(specs, device, replicas: int) -> PeerBuffers:
    """Fan-out onto `replicas` buffers of this GPU (destination 0 is the engine's own): the
    single-GPU stand-in for peers, used by the tests and the single-GPU bench."""
    _, _, nc, ns = _layout(specs)
    cs = [torch.zeros(nc, dtype=torch.uint8, device=device) for _ in range(replicas)]
    ss = [torch.zeros(ns, dtype=torch.float32, device=device) for _ in range(replicas)]
    return PeerBuffers(cs[0], ss[0], [c.data_ptr() - cs[0].data_ptr() for c in cs],
                       [x.data_ptr() - ss[0].data_ptr() for x in ss], keep=(cs, ss))


def symmetric_peer_buffers(specs, device, group=None) -> PeerBuffers:
    """Engine buffers in torch symmetric memory: every rank's buffer is mapped into every other
    rank's address space over NVLink, so the fan-out deltas are peer base - local base.  The
    fence is the symmetric-memory barrier (all ranks' stores done before anyone reads)."""
    import torch.distributed._symmetric_memory as symm_mem
    _, _, nc, ns = _layout(specs)
    group = group or dist.group.WORLD
    c = symm_mem.empty(nc, dtype=torch.uint8, device=device)
    s = symm_mem.empty(ns, dtype=torch.float32, device=device)
    hc = symm_mem.rendezvous(c, group)
    hs = symm_mem.rendezvous(s, group)
    cd = [p - c.data_ptr() for p in hc.buffer_ptrs]
    sd = [p - s.data_ptr() for p in hs.buffer_ptrs]
    return PeerBuffers(c, s, cd, sd, fence=lambda: hc.barrier(), keep=(c, s, hc, hs))


def _default_quantize(w: torch.Tensor, codes: torch.Tensor, scales: torch.Tensor, flag=None) -> None:
    from .fp8q import quantize_weight_blockwise
    quantize_weight_blockwise(w, codes, scales, nonfinite_flag=flag)


class WeightSyncEngine:
    """Persistent FP8 engine buffers (codes + scales) for a set of weights, refreshed every
    RL step from this rank's BF16 shards (versioned snapshot, stale-step
    rejection, post-state equals quantize(snapshot) bitwise)."""

    def __init__(self, specs: Sequence[TensorSpec], device, group=None,
                 quantize_fn: Optional[QuantizeFn] = None, peers: Optional[PeerBuffers] = None):
        self.specs = list(specs)
        self.peers = peers
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.device = torch.device(device)
        self.quantize_fn = quantize_fn or _default_quantize
        self.plans: Dict[str, List[Shard]] = {s.name: plan_shards(s, self.world) for s in self.specs}
        self.codes: Dict[str, torch.Tensor] = {}
        self.scales: Dict[str, torch.Tensor] = {}
        if peers is not None:
            co, so, _, _ = _layout(self.specs)
            for s in self.specs:
                self.codes[s.name] = peers.codes_flat[co[s.name]:co[s.name] + s.rows * s.k].view(s.rows, s.k)
                nsc = s.scale_rows * s.scale_cols
                self.scales[s.name] = peers.scales_flat[so[s.name]:so[s.name] + nsc].view(s.scale_rows, s.scale_cols)
        else:
            for s in self.specs:
                self.codes[s.name] = torch.empty((s.rows, s.k), dtype=torch.uint8, device=self.device)
                self.scales[s.name] = torch.empty((s.scale_rows, s.scale_cols), dtype=torch.float32,
                                                  device=self.device)
        self.loaded_step = -1
        # device int32, set by every quantizer launch that meets a NaN/Inf (fp8q.h contract);
        # read before loaded_step advances (strict) or by check_finite() (deferred)
        self.nonfinite = torch.zeros(1, dtype=torch.int32, device=self.device) \
            if self.device.type == "cuda" else None
        self.poisoned = False

    def my_shard(self, name: str) -> Shard:
        return self.plans[name][self.rank]

    def shard_rows(self, name: str) -> Tuple[int, int]:
        sh = self.my_shard(name)
        return sh.row0, sh.row1

    def quantize_local(self, name: str, w_shard: torch.Tensor) -> None:
        """Quantize this rank's BF16 shard straight into its slot of the full buffers."""
        sh = self.my_shard(name)
        if w_shard.shape[0] != sh.row1 - sh.row0:
            raise ValueError(f"{name}: shard has {w_shard.shape[0]} rows, plan says {sh.row1 - sh.row0}")
        self.quantize_fn(w_shard, self.codes[name][sh.row0:sh.row1], self.scales[name][sh.srow0:sh.srow1])

    def gather(self, name: str, async_op: bool = False):
        """In-place all-gather of codes and scales: every rank ends with the full FP8 weight."""
        if self.world == 1:
            return []
        sh = self.my_shard(name)
        c, s = self.codes[name], self.scales[name]
        h1 = dist.all_gather_into_tensor(c, c[sh.row0:sh.row1], group=self.group, async_op=async_op)
        h2 = dist.all_gather_into_tensor(s, s[sh.srow0:sh.srow1], group=self.group, async_op=async_op)
        return [h for h in (h1, h2) if h is not None]

    def gather_many(self, names: Sequence[str]) -> None:
        """All-gathers of several tensors as ONE grouped NCCL call (one launch for the whole
        bucket instead of two per tensor); backends without coalescing (gloo) loop."""
        if self.world == 1 or not names:
            return
        backend = dist.get_backend(self.group)
        if backend == "nccl":
            with dist._coalescing_manager(group=self.group, device=self.device):
                for n in names:
                    self.gather(n)
        else:
            for n in names:
                self.gather(n)

    def _validate(self, shards: Dict[str, torch.Tensor]) -> None:
        """Every shard's presence, shape, dtype and device, checked before anything is launched
        or any collective is entered, so a bad shard never leaves a half-synced engine (or a
        rank that skips collectives its peers are blocked in)."""
        missing = [s.name for s in self.specs if s.name not in shards]
        if missing:
            raise KeyError(f"missing shards: {missing}")
        for s in self.specs:
            sh = self.my_shard(s.name)
            w = shards[s.name]
            want = (sh.row1 - sh.row0, s.k)
            if tuple(w.shape) != want:
                raise ValueError(f"{s.name}: shard shape {tuple(w.shape)}, plan says {want}")
            if w.dtype != torch.bfloat16:
                raise ValueError(f"{s.name}: shard dtype {w.dtype}, expected torch.bfloat16")
            if w.device != self.codes[s.name].device:
                raise ValueError(f"{s.name}: shard on {w.device}, engine buffers on {self.codes[s.name].device}")

    def _local_items(self, specs, shards):
        items = []
        for s in specs:
            sh = self.my_shard(s.name)
            items.append((shards[s.name], self.codes[s.name][sh.row0:sh.row1],
                          self.scales[s.name][sh.srow0:sh.srow1]))
        return items

    def check_finite(self) -> None:
        """Deferred non-finite check (for sync_step(strict=False)): raises NonFiniteWeightError
        if any quantizer launch since the last check met a NaN/Inf, on every rank alike (the
        flag is MAX-reduced over the group), and re-arms the flag.  Host-synchronising."""
        if self.nonfinite is None:
            return
        f = self.nonfinite.clone()
        if self.world > 1:
            dist.all_reduce(f, op=dist.ReduceOp.MAX, group=self.group)
        bad = int(f.item()) != 0
        self.nonfinite.zero_()
        if bad:
            self.poisoned = True
            raise NonFiniteWeightError("non-finite BF16 weight in a synced shard; engine buffers undefined")

    def sync_step(self, step: int, shards: Dict[str, torch.Tensor], comm_stream=None,
                  bucket: int = 16, ready=None, on_bucket=None, strict: bool = True) -> None:
        """One weight synchronisation: quantize every local shard, all-gather.

        Buckets of `bucket` tensors: one batched quantizer launch per bucket, then one grouped
        all-gather of that bucket -- on `comm_stream` when given, so bucket i's gather overlaps
        bucket i+1's quantization on the compute stream.  `ready` (name -> CUDA event): a
        bucket's quantization first waits for its tensors' events (e.g. their host uploads), so
        small buckets pipeline with the uploads; `on_bucket(names)` is called on the stream that
        finished a bucket (after its gather), e.g. to record an event a consumer waits on.

        Non-finite input sets the engine's device flag in the quantizer.  strict:
        the flag is read (MAX over ranks) before `loaded_step` advances -- a host sync -- and a
        NonFiniteWeightError leaves `loaded_step` unchanged.  strict=False: no host sync; call
        check_finite() later (the flag accumulates until then)."""
        if step <= self.loaded_step:
            raise StaleStepError(f"step {step} is not newer than loaded step {self.loaded_step}")
        self._validate(shards)
        flag = self.nonfinite
        if strict and flag is not None:
            flag.zero_()
        if self.peers is not None:
            # NEXT-1: the quantizer writes every rank's buffer itself; no gather pass.  The
            # opening fence keeps a fast rank from overwriting a peer's step-t weights while the
            # peer may still be reading them; the closing fence publishes every rank's stores.
            from .fp8q import quantize_weight_blockwise_fanout
            self.peers.fence()
            for b0 in range(0, len(self.specs), bucket):
                quantize_weight_blockwise_fanout(self._local_items(self.specs[b0:b0 + bucket], shards),
                                                 self.peers.codes_delta, self.peers.scales_delta,
                                                 nonfinite_flag=flag)
            self.peers.fence()
            self._commit(step, strict)
            return
        batched = self.quantize_fn is _default_quantize
        if batched:
            from .fp8q import quantize_weight_blockwise_batched
        overlap = comm_stream is not None and self.world > 1
        compute = torch.cuda.current_stream(self.device) if overlap else None
        for b0 in range(0, len(self.specs), bucket):
            chunk = self.specs[b0:b0 + bucket]
            if ready is not None:
                cs = torch.cuda.current_stream(self.device)
                for sp in chunk:
                    if sp.name in ready:
                        cs.wait_event(ready[sp.name])
            if batched:
                quantize_weight_blockwise_batched(self._local_items(chunk, shards), nonfinite_flag=flag)
            else:
                for s in chunk:
                    self.quantize_local(s.name, shards[s.name])
            names = [s.name for s in chunk]
            if overlap:
                ev = torch.cuda.Event()
                ev.record(compute)
                with torch.cuda.stream(comm_stream):
                    comm_stream.wait_event(ev)
                    self.gather_many(names)
                    if on_bucket is not None:
                        on_bucket(names)
            else:
                self.gather_many(names)
                if on_bucket is not None:
                    on_bucket(names)
        if overlap:
            compute.wait_stream(comm_stream)
        self._commit(step, strict)

    def _commit(self, step: int, strict: bool) -> None:
        if strict:
            self.check_finite()
        self.poisoned = False
        self.loaded_step = step
