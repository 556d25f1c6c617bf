// gemm.cu -- blockwise-scaled FP8 GEMM for sm_100a (tcgen05 + TMA + TMEM), dense and grouped.
//
// Computes ("W8A8 ... DeepGEMM"; granularity PAPER.md:233)
//     D[m,n] = sum_kb  (sa[kb][m] * sb[n/128][kb]) * P_kb[m,n],
//     P_kb[m,n] = sum_{k in kb} dec(a[m,k]) * dec(b[n,k])      (128-deep k-block kb)
// The scales are arbitrary fp32 (amax/448), so they cannot ride in the tensor core's UE8M0
// block-scale path: every k-block's partial P_kb is produced by the tensor core in TMEM and
// promoted by CUDA-core FMAs into an fp32 register accumulator ("scale promotion").
//
// CTA = 12 warps (3 warpgroups), persistent over 128x256 output tiles (M-fastest order so
// concurrent CTAs share B tiles and the whole A panel stays L2-resident).  Warpgroup 0 gives
// registers away (setmaxnreg.dec 72) and warpgroups 1-2 take them (setmaxnreg.inc 216): the
// register file is per SM sub-partition, so 3 warps x 168 at launch become 72 + 216 + 216 (the CTA pool: 128 x 96 released = 256 x 48 taken).
//   warp 0        TMA producer: per k-block, A 128x128 B and B 256x128 B into a 4-stage ring
//                 (128-byte swizzle), mbarrier full/empty handshake with the MMA warp.
//   warp 1        TMEM owner (512 columns) and MMA issuer: 4 x tcgen05.mma.kind::f8f6f4
//                 (M=128, N=256, K=32) per k-block into TMEM buffer (it % 2), fresh
//                 accumulation per k-block; tcgen05.commit frees the smem stage and
//                 publishes the partial.
//   warps 2,3     idle (they only donate registers).
//   warps 4..11   promotion/epilogue: warp w reads TMEM lanes 32*(w%4)..+31 (its 32 rows),
//                 warps 4-7 columns 0-127 and 8-11 columns 128-255 (one weight n-block each,
//                 so one scale product per thread per k-block).  acc += P_kb * (sa*sb) with
//                 packed FFMA2; the TMEM buffer is released as soon as it is read, so the
//                 tensor core fills the other buffer while the FMAs run.  After the last
//                 k-block each thread writes its row segment (BF16 = RNE of the F32 value).
// Determinism: fixed k-block order, no atomics.  DESIGN.md §5.2 has the roofline analysis.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "ptx.cuh"
#include "quant_kernels.h"

namespace fp8q {
namespace {

constexpr int BM = 128;
constexpr int BK = 128;
constexpr int A_TILE = BM * BK;  // bytes (E4M3)
constexpr int NUM_THREADS = 384;
constexpr int EPI_WARP0 = 4;
constexpr int TMEM_COLS = 512;
constexpr int NUM_EPI_WARPS = 8;
constexpr int RASTER_GM = 16;  // m-tiles per raster band
// operand stages: 160 KB + the 64 KB BF16 epilogue staging + barriers + alignment slack = the
// 227 KB per-CTA limit (a 6th pair stage does not fit: measured, launch rejected)
constexpr int SMEM_BUDGET = 160 * 1024;
// Output staging for the TMA-store epilogue: per promotion warp four 32-row x 64-byte
// chunks (2 KB each, 64-byte swizzle) -> 8 warps x 8 KB.  A BF16 half-tile row segment
// (128 columns) is exactly 4 chunks, so a tile's stores never wait for each other.
constexpr int kSmemGroups = 512;  // groups whose offsets the one-CTA kernel stages in smem
constexpr int EPI_CHUNKS = 4;
constexpr int EPI_CHUNK_BYTES = 32 * 64;
constexpr int EPI_STAGE_BYTES = NUM_EPI_WARPS * EPI_CHUNKS * EPI_CHUNK_BYTES;
// setmaxnreg budget: the CTA's register pool is fixed at launch (384 threads x 168), so what
// warpgroup 0 releases must cover what warpgroups 1-2 take, or setmaxnreg.inc never returns.
constexpr int REGS_LAUNCH = 168;
constexpr int REGS_CTRL = 72;
constexpr int REGS_EPI = 216;
static_assert(128 * (REGS_LAUNCH - REGS_CTRL) >= 256 * (REGS_EPI - REGS_LAUNCH), "register pool overdrawn");

// Tile configuration.  BN = 256: 2 TMEM partial buffers, 4 smem stages, 128 accumulator
// registers per promotion thread.  BN = 128: 4 TMEM partial buffers (the tensor core can run
// 3 k-blocks ahead of the promotion warps), 6 smem stages, 64 accumulators per thread.
template <int BN_>
struct Cfg {
    static constexpr int BN = BN_;
    static constexpr int B_TILE = BN * BK;
    static constexpr int STAGE_BYTES = A_TILE + B_TILE;
    static constexpr int STAGES = SMEM_BUDGET / STAGE_BYTES;
    static constexpr int TMEM_BUFS = TMEM_COLS / BN;
    static constexpr int EPI_COLS = BN / 2;  // columns per promotion thread
    static constexpr uint32_t IDESC = idesc_e4m3_f32(BM, BN);
    static constexpr size_t SMEM_BYTES = 1024 + size_t(STAGES) * STAGE_BYTES + EPI_STAGE_BYTES + 512;
};

struct KParams {
    const float* sa;
    int64_t ld_sa;
    const float* sb;
    int64_t ld_sb;
    int64_t stride_sb;
    void* d;
    int64_t ld_d;
    int out_f32;
    int64_t m;
    int64_t n;
    int num_kb;
    int num_n_tiles;
    const int32_t* offsets;  // nullptr: one group of m rows
    int splits;              // split-K slices per tile (one-CTA kernel, dense, small M); 1 = off
    int raster;              // m-tiles per raster band (TileCursor); < 0: -(n-tiles per band), n fastest
    float* ws;               // split-K partials [tile][split][128][BN] fp32
    int32_t* counters;       // split-K arrival counters [tile], zero between launches
    int groups;
    int dp_tiles;            // tiles [0, dp_tiles) whole, the rest in `splits` K slices
    int fix_bulk;            // split fixup through the idle smem ring (each CTA's last item only)
};

// Walks the (group, m-tile, n-tile) sequence; t must increase between calls.  TM = rows per
// tile (128 for one CTA, 256 for a CTA pair), GM = m-tiles per raster band.
template <int TM, int GM_UNUSED>
struct TileCursor {
    // 32-bit tile arithmetic on purpose: 64-bit division is a ~100-instruction software
    // routine, and this runs between tiles on the promotion warps' critical path.
    int g;
    int base;    // first linear tile index of group g
    int row0;    // first A/D row of group g
    int rows;    // rows in group g
    int mtiles;  // ceil(rows / TM)
    const int32_t* offs;  // the group offsets: a shared-memory copy when the kernel made one
    __device__ void load(const KParams& p) {
        if (p.offsets != nullptr) {
            row0 = offs[g];
            rows = offs[g + 1] - row0;
        } else {
            row0 = 0;
            rows = static_cast<int>(p.m);
        }
        mtiles = (rows + TM - 1) / TM;
    }
    __device__ void init(const KParams& p, const int32_t* smem_offs = nullptr) {
        g = 0;
        base = 0;
        offs = smem_offs != nullptr ? smem_offs : p.offsets;
        if (p.groups > 0) load(p);
    }
    // Returns false when t is past the last tile.
    __device__ bool seek(const KParams& p, int t, int& mt, int& nt) {
        if (g >= p.groups) return false;
        while (t >= base + mtiles * p.num_n_tiles) {
            base += mtiles * p.num_n_tiles;
            if (++g >= p.groups) return false;
            load(p);
        }
        // Grouped raster: bands of GM m-tiles; inside a band m is fastest, so the ~148
        // concurrent tiles cover a compact RASTER_GM x ~9 block of the output and both the A
        // band and the B tiles they touch stay L2-resident (K = 12288 would otherwise re-read A).
        const unsigned l = static_cast<unsigned>(t - base);
        if (p.raster < 0) {  // B-resident raster: bands of -raster n-tiles, n fastest inside
            const unsigned GN = static_cast<unsigned>(-p.raster);
            const unsigned nt_all = static_cast<unsigned>(p.num_n_tiles);
            const unsigned spn = GN * static_cast<unsigned>(mtiles);
            const unsigned bn = l / spn;
            const unsigned rn = l - bn * spn;
            const unsigned gn = min(GN, nt_all - bn * GN);
            const unsigned qn = rn / gn;
            nt = static_cast<int>(bn * GN + (rn - qn * gn));
            mt = static_cast<int>(qn);
            return true;
        }
        const unsigned GM = static_cast<unsigned>(p.raster);
        const unsigned span = GM * static_cast<unsigned>(p.num_n_tiles);
        const unsigned band = l / span;
        const unsigned r = l - band * span;
        const unsigned gm = min(GM, static_cast<unsigned>(mtiles) - band * GM);
        const unsigned q = r / gm;
        mt = static_cast<int>(band * GM + (r - q * gm));
        nt = static_cast<int>(q);
        return true;
    }
};

__device__ __forceinline__ void ffma2(float2& acc, const float2 v, const float f) {
    uint64_t a = *reinterpret_cast<uint64_t*>(&acc);
    const uint64_t x = *reinterpret_cast<const uint64_t*>(&v);
    const float2 ff = make_float2(f, f);
    const uint64_t s = *reinterpret_cast<const uint64_t*>(&ff);
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a) : "l"(x), "l"(s));
    acc = *reinterpret_cast<float2*>(&a);
}

// One output tile's promotion + store, for one promotion thread: its row `row`, columns
// [col0, col0 + EPI_COLS).  For every k-block: wait for the partial in TMEM buffer it % NBUF,
// tcgen05.ld it, hand the buffer back (to the leader CTA of a pair when PAIR), and
// acc += P_kb * (sa[kb][row] * sb[col0/128][kb]) with packed FFMA2.
// One promotion thread's share of an output tile: row `row`, columns [col0, col0 + BN/2).
struct EpiTile {
    int64_t row;      // this thread's output row
    int64_t row_end;  // end of the rows this tile may write (group end / m)
    int64_t col0;     // first of this thread's columns
    int g;            // group (MoE expert) index
    int kb0, kb1;     // this work item's k-block range
    int tile;         // split-K workspace tile index (pair: local split tile * 2 + CTA rank)
    int split;        // split-K slice of this work item
    int nsplit;       // K slices of this tile (1: whole tile, stored directly)
};
// The first two k-blocks' (sa, sb) of a tile: loaded one tile ahead so the HBM/L2 latency of
// the first scales overlaps the previous tile's last k-blocks and stores.
struct ScalePre {
    float sa0, sb0, sa1, sb1;
};
__device__ __forceinline__ bool tile_live(const KParams& p, const EpiTile& t) {
    return t.row < t.row_end && t.col0 < p.n;
}
// Where a tile's first two k-blocks' scales live (computed once, so only two pointers and a
// flag -- not the whole next tile -- stay live across the k-loop).
struct ScalePtrs {
    const float* sap;
    const float* sbp;
    int64_t ld_sa;
    bool live;
    bool two;
};
__device__ __forceinline__ ScalePtrs scale_ptrs(const KParams& p, const EpiTile& t) {
    ScalePtrs q;
    q.live = tile_live(p, t);
    q.two = t.kb1 - t.kb0 > 1;
    q.ld_sa = p.ld_sa;
    q.sap = p.sa + t.row + int64_t(t.kb0) * p.ld_sa;
    q.sbp = p.sb + int64_t(t.g) * p.stride_sb + (t.col0 / 128) * p.ld_sb + t.kb0;
    return q;
}
__device__ __forceinline__ ScalePre load_scales(const ScalePtrs& q) {
    ScalePre s{0.f, 0.f, 0.f, 0.f};
    if (q.live) {
        s.sa0 = __ldg(q.sap);
        s.sb0 = __ldg(q.sbp);
        if (q.two) {
            s.sa1 = __ldg(q.sap + q.ld_sa);
            s.sb1 = __ldg(q.sbp + 1);
        }
    }
    return s;
}
__device__ __forceinline__ ScalePre prefetch_scales(const KParams& p, const EpiTile& t) {
    return load_scales(scale_ptrs(p, t));
}

__device__ __forceinline__ int split_begin(const KParams& p, int s) {
    return (s * p.num_kb) / p.splits;  // 32-bit: s * num_kb < 2^31 for any real K
}

// Work item v (split plans: plan_split): below dp_tiles the whole tile v;
// past it slice sp of tile dp_tiles + (v - dp_tiles) / splits.  Returns the tile index (past
// the last tile when v is), its k-block range in [kb0, kb1).
__device__ __forceinline__ int work_item(const KParams& p, int v, int& sp, int& kb0, int& kb1) {
    if (v < p.dp_tiles) {
        sp = 0;
        kb0 = 0;
        kb1 = p.num_kb;
        return v;
    }
    const int u = v - p.dp_tiles;
    const int tq = u / p.splits;
    sp = u - tq * p.splits;
    kb0 = split_begin(p, sp);
    kb1 = split_begin(p, sp + 1);
    return p.dp_tiles + tq;
}

// For every k-block: wait for the partial in TMEM buffer it % NBUF, tcgen05.ld it, hand the
// buffer back (to the leader CTA of a pair when PAIR), and
// acc += P_kb * (sa[kb][row] * sb[col0/128][kb]) with packed FFMA2; then store the tile.
template <int BN, int NBUF, bool PAIR>
__device__ __forceinline__ void promote_tile(const KParams& p, const CUtensorMap* tmD, uint8_t* stg,
                                             uint8_t* ring, uint64_t* fixbar,
                                             const EpiTile& tile, const ScalePre& pre, bool has_next,
                                             const EpiTile& next, ScalePre& next_pre, uint32_t tmem,
                                             int qd, int h, int lane, uint64_t* tfull,
                                             uint64_t* tempty, uint32_t& it, uint64_t* stg_full,
                                             uint64_t* stg_empty, uint32_t& tile_no) {
    constexpr int EPI_COLS = BN / 2;
    constexpr int CHUNKS = EPI_COLS / 32;  // tcgen05.ld 32x32b.x32 per promotion thread
    static_assert(EPI_COLS / 32 <= EPI_CHUNKS, "BF16 row segment must fit the staging chunks");
    const int64_t row = tile.row;
    const int64_t row_end = tile.row_end;
    const int64_t col0 = tile.col0;
    const bool live = tile_live(p, tile);
    const float* sap = p.sa + row;
    const float* sbp = p.sb + int64_t(tile.g) * p.stride_sb + (col0 / 128) * p.ld_sb;
    float2 acc[EPI_COLS / 2];
#pragma unroll
    for (int j = 0; j < EPI_COLS / 2; ++j) acc[j] = make_float2(0.f, 0.f);
    // Scale prefetch two k-blocks ahead; the raw values are only multiplied when used,
    // so the load latency never sits between the TMEM-full wait and the FMAs.
    float sa0 = pre.sa0, sb0 = pre.sb0, sa1 = pre.sa1, sb1 = pre.sb1;
    ScalePtrs nq = scale_ptrs(p, next);
    nq.live = nq.live && has_next;
    const int kb0 = tile.kb0, kb1 = tile.kb1;
    for (int kb = kb0; kb < kb1; ++kb, ++it) {
        const float f = sa0 * sb0;
        sa0 = sa1;
        sb0 = sb1;
        if (live && kb + 2 < kb1) {
            sa1 = __ldg(sap + int64_t(kb + 2) * p.ld_sa);
            sb1 = __ldg(sbp + kb + 2);
        }
        if (kb == (kb1 - kb0 > 4 ? kb1 - 4 : kb0)) next_pre = load_scales(nq);
        const uint32_t buf = it % NBUF;
        const uint32_t bph = (it / NBUF) & 1u;
        mbar_wait(&tfull[buf], bph);
        tc_fence_after();
        const uint32_t taddr = tmem + (static_cast<uint32_t>(qd * 32) << 16) + buf * BN + h * EPI_COLS;
        // Software-pipelined: the tcgen05.ld of chunk c+1 is in flight while chunk c's FMAs
        // issue, so each TMEM load latency after the first overlaps useful work.
        float v[2][32];
        tmem_ld_32x32b_x32(taddr, v[0]);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < CHUNKS; ++c) {
            if (c + 1 < CHUNKS) tmem_ld_32x32b_x32(taddr + (c + 1) * 32, v[(c + 1) & 1]);
#pragma unroll
            for (int j = 0; j < 16; ++j)
                ffma2(acc[c * 16 + j], make_float2(v[c & 1][2 * j], v[c & 1][2 * j + 1]), f);
            if (c + 1 < CHUNKS) tmem_wait_ld();
            if (c + 2 == CHUNKS || CHUNKS == 1) {  // last chunk loaded: hand the buffer back
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (PAIR)
                        mbar_arrive_cluster(&tempty[buf], 0);
                    else
                        mbar_arrive(&tempty[buf]);
                }
            }
        }
    }
    if (tile.nsplit > 1) {
        // ---- split-K: park this slice's fp32 partial; the last slice to arrive sums all
        // slices in slice order (deterministic) and stores the tile.  Layout per (tile, slice):
        // [column half h][16-byte unit j][row] -- a warp's access to unit j covers its 32
        // consecutive rows, 512 contiguous bytes.  (Row-major partials, each lane 1 KB from the
        // next, made the fixup ~4x slower than the k-loop it split: 32 sectors per instruction.)
        __shared__ int sk_last;
        constexpr int UNITS = EPI_COLS / 4;  // 16-byte units per thread
        const int r_in = qd * 32 + lane;     // row within the tile
        float4* mine = reinterpret_cast<float4*>(p.ws) +
                       ((tile.tile * tile.nsplit + tile.split) * 2 + h) * UNITS * BM + r_in;
        if (live) {  // only real rows/columns are parked and summed (decode: M << 128)
#pragma unroll
            for (int j = 0; j < UNITS; ++j)
                st_v4(mine + j * BM, __float_as_uint(acc[2 * j].x), __float_as_uint(acc[2 * j].y),
                      __float_as_uint(acc[2 * j + 1].x), __float_as_uint(acc[2 * j + 1].y));
        }
        __threadfence();
        asm volatile("bar.sync 1, %0;" ::"n"(NUM_EPI_WARPS * 32) : "memory");
        if (threadIdx.x == EPI_WARP0 * 32) {
            const int old = atomicAdd(&p.counters[tile.tile], 1);
            __threadfence();
            sk_last = (old == tile.nsplit - 1);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(NUM_EPI_WARPS * 32) : "memory");
        if (!sk_last) return;
        if (p.fix_bulk) {
            // This slice was the CTA's last work item and its MMAs have completed, so the
            // shared-memory ring is idle: bulk-copy each slice's 64 KB column half into it (one
            // copy in flight per half, issued by the half's first warp) and add from shared
            // memory -- the register path below keeps only ~16 loads per thread in flight and
            // is bound by L2 latency.
            constexpr uint32_t HALF_BYTES = UNITS * BM * 16;
            uint8_t* buf = ring + h * HALF_BYTES;
            const float4* src = reinterpret_cast<const float4*>(p.ws) + (tile.tile * tile.nsplit * 2 + h) * UNITS * BM;
            const bool issuer = qd == 0 && lane == 0;
            if (issuer) fence_proxy_async_global();
#pragma unroll
            for (int j = 0; j < EPI_COLS / 2; ++j) acc[j] = make_float2(0.f, 0.f);
            for (int sl = 0; sl < tile.nsplit; ++sl) {
                if (issuer) {
                    mbar_arrive_expect_tx(&fixbar[h], HALF_BYTES);
                    bulk_load_g2s(smem_u32(buf), src + sl * 2 * UNITS * BM, HALF_BYTES, &fixbar[h]);
                }
                mbar_wait(&fixbar[h], static_cast<uint32_t>(sl) & 1u);
                const uint32_t rb = smem_u32(buf) + static_cast<uint32_t>(r_in) * 16u;
#pragma unroll
                for (int j = 0; j < UNITS; ++j) {
                    uint32_t x0, x1, x2, x3;
                    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3)
                                 : "r"(rb + static_cast<uint32_t>(j * BM) * 16u));
                    acc[2 * j].x += __uint_as_float(x0);
                    acc[2 * j].y += __uint_as_float(x1);
                    acc[2 * j + 1].x += __uint_as_float(x2);
                    acc[2 * j + 1].y += __uint_as_float(x3);
                }
                // the half's 4 warps are done with buf before the next slice overwrites it
                asm volatile("bar.sync %0, 128;" ::"r"(2 + h) : "memory");
            }
            if (threadIdx.x == EPI_WARP0 * 32) p.counters[tile.tile] = 0;  // reusable workspace
        } else {
        const float4* base = reinterpret_cast<const float4*>(p.ws) + (tile.tile * tile.nsplit * 2 + h) * UNITS * BM + r_in;
#pragma unroll
        for (int j = 0; j < EPI_COLS / 2; ++j) acc[j] = make_float2(0.f, 0.f);
        for (int sl = 0; sl < tile.nsplit && live; ++sl) {
            const float4* src = base + sl * 2 * UNITS * BM;
#pragma unroll
            for (int j = 0; j < UNITS; ++j) {
                const float4 v = __ldcg(src + j * BM);
                acc[2 * j].x += v.x;
                acc[2 * j].y += v.y;
                acc[2 * j + 1].x += v.z;
                acc[2 * j + 1].y += v.w;
            }
        }
        if (threadIdx.x == EPI_WARP0 * 32) p.counters[tile.tile] = 0;  // reusable workspace
        }
    }
    if (col0 >= p.n) return;  // warp-uniform: these columns are past the matrix
    // ---- output: the warp's 32 rows x EPI_COLS columns, through the warp's smem staging:
    // each lane writes its row as 64-byte-swizzled 16 B units (conflict-free), then the warp
    // reads the staging back row-contiguously so every STG.128 instruction writes two full
    // 256-byte row segments (coalesced; rows past row_end and columns past n are masked, which
    // also covers MoE group tails).  Plain loads/stores: no async-proxy fence, no TMA queue.
    (void)tmD;
    const int64_t row_base = row - lane;
    if (!p.out_f32 && tile.nsplit == 1 && EPI_COLS * 2 == 4 * 64) {  // must match the store-warp role
        // BF16 production path: park the row segment in this warp's staging (64-byte swizzled
        // 16 B units, conflict-free) and hand it to the store warp of this column half, which
        // writes it to global memory while this warp already promotes the next tile.
        const uint32_t ph = tile_no & 1u;
        ++tile_no;
        mbar_wait(&stg_empty[h], ph ^ 1u);  // the store warp drained this staging (a tile ago)
        const uint32_t swz = static_cast<uint32_t>((lane >> 1) & 3);
        const uint32_t stg_base = smem_u32(stg);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const uint32_t base = stg_base + c * EPI_CHUNK_BYTES + lane * 64;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                uint32_t w[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float2 a = acc[c * 16 + j * 4 + e];
                    __nv_bfloat162 b2 = __floats2bfloat162_rn(a.x, a.y);
                    w[e] = *reinterpret_cast<uint32_t*>(&b2);
                }
                st_shared_v4(base + 16u * (static_cast<uint32_t>(j) ^ swz), w[0], w[1], w[2], w[3]);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&stg_full[h]);  // release: the staging writes above
        return;
    }
    // a split tile after whole ones: the store warp may still be draining this
    // warp's staging from the last parked tile
    if (tile_no > 0) mbar_wait(&stg_empty[h], (tile_no - 1) & 1u);
    const uint32_t swz = static_cast<uint32_t>((lane >> 1) & 3);
    const uint32_t stg_base = smem_u32(stg);
    // One staging pass: CH chunks of 32 rows x 64 B (CH = 4 -> 256 B row segments, 16 lanes
    // per row; CH = 2 -> 128 B, 8 lanes per row).
    auto drain = [&](int64_t gcol0_bytes, int esz, auto ch_tag) {
        constexpr int CH = decltype(ch_tag)::value;
        constexpr int UPR = CH * 4;        // 16 B units per row segment
        constexpr int RPI = 32 / UPR;      // rows per warp instruction
        __syncwarp();
        char* dbase = static_cast<char*>(p.d);
#pragma unroll
        for (int i = 0; i < 32 / RPI; ++i) {
            const int r = RPI * i + lane / UPR;
            const int u = lane % UPR;
            const uint32_t src = stg_base + (u >> 2) * EPI_CHUNK_BYTES + r * 64 +
                                 16u * (static_cast<uint32_t>(u & 3) ^ static_cast<uint32_t>((r >> 1) & 3));
            uint32_t x0, x1, x2, x3;
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3) : "r"(src));
            const int64_t grow = row_base + r;
            const int64_t gbyte = gcol0_bytes + 16 * u;
            if (grow < row_end && gbyte < p.n * esz)
                st_v4(dbase + grow * p.ld_d * esz + gbyte, x0, x1, x2, x3);
        }
        __syncwarp();
    };
    if (p.out_f32) {
        constexpr int CH = EPI_COLS * 4 >= 256 ? 4 : 2;  // chunks per pass
        constexpr int PASS_COLS = CH * 16;               // fp32 columns per pass
#pragma unroll
        for (int pass = 0; pass < EPI_COLS / PASS_COLS; ++pass) {
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const uint32_t base = stg_base + c * EPI_CHUNK_BYTES + lane * 64;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int a = pass * (PASS_COLS / 2) + c * 8 + j * 2;
                    st_shared_v4(base + 16u * (static_cast<uint32_t>(j) ^ swz), __float_as_uint(acc[a].x),
                                 __float_as_uint(acc[a].y), __float_as_uint(acc[a + 1].x),
                                 __float_as_uint(acc[a + 1].y));
                }
            }
            drain((col0 + pass * PASS_COLS) * 4, 4, std::integral_constant<int, CH>{});
        }
    } else {
        constexpr int CH = EPI_COLS * 2 >= 256 ? 4 : 2;
        constexpr int PASS_COLS = CH * 32;  // bf16 columns per pass
#pragma unroll
        for (int pass = 0; pass < EPI_COLS / PASS_COLS; ++pass) {
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const uint32_t base = stg_base + c * EPI_CHUNK_BYTES + lane * 64;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    uint32_t w[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float2 a = acc[pass * (PASS_COLS / 2) + c * 16 + j * 4 + e];
                        __nv_bfloat162 b2 = __floats2bfloat162_rn(a.x, a.y);
                        w[e] = *reinterpret_cast<uint32_t*>(&b2);
                    }
                    st_shared_v4(base + 16u * (static_cast<uint32_t>(j) ^ swz), w[0], w[1], w[2], w[3]);
                }
            }
            drain((col0 + pass * PASS_COLS) * 2, 2, std::integral_constant<int, CH>{});
        }
    }
}

// Store warp (warps 2 and 3, otherwise idle): for every tile, wait until the 4 promotion
// warps of column half h have parked their 32 x 128 BF16 slices, copy the 4 slices to global
// memory with coalesced STG.128 (two full 256-byte row segments per instruction; rows past
// row_end / columns past n masked), then release the staging.
__device__ __forceinline__ void store_tile_half(const KParams& p, const uint8_t* smEpi, int h, int lane,
                                                int64_t row0_tile, int64_t row_end, int64_t col0,
                                                uint64_t* stg_full, uint64_t* stg_empty, uint32_t& tile_no) {
    const uint32_t ph = tile_no & 1u;
    ++tile_no;
    mbar_wait(&stg_full[h], ph);
    char* dbase = static_cast<char*>(p.d);
#pragma unroll 1
    for (int q = 0; q < 4; ++q) {  // slice of promotion warp EPI_WARP0 + 4h + q (TMEM quarter q)
        const uint32_t sbase = smem_u32(smEpi + (4 * h + q) * EPI_CHUNKS * EPI_CHUNK_BYTES);
        const int64_t rbase = row0_tile + q * 32;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int r = 2 * i + (lane >> 4);
            const int u = lane & 15;
            const uint32_t src = sbase + (u >> 2) * EPI_CHUNK_BYTES + r * 64 +
                                 16u * (static_cast<uint32_t>(u & 3) ^ static_cast<uint32_t>((r >> 1) & 3));
            uint32_t x0, x1, x2, x3;
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3) : "r"(src));
            const int64_t grow = rbase + r;
            const int64_t gcol = col0 + 8 * u;
            if (grow < row_end && gcol < p.n)
                st_v4(dbase + (grow * p.ld_d + gcol) * 2, x0, x1, x2, x3);
        }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&stg_empty[h]);
}

template <int BN_>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    fp8_block_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                          const __grid_constant__ CUtensorMap tmB,
                          const __grid_constant__ CUtensorMap tmD, const KParams p) {
    using C = Cfg<BN_>;
    constexpr int BN = C::BN;
    constexpr int STAGES = C::STAGES;
    constexpr int NBUF = C::TMEM_BUFS;
    constexpr int EPI_COLS = C::EPI_COLS;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint8_t* smA = smem;
    uint8_t* smB = smem + STAGES * A_TILE;
    uint8_t* smEpi = smem + STAGES * C::STAGE_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(smEpi + EPI_STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + NBUF;
    uint64_t* stg_full = tempty + NBUF;   // [2]: per column half, 4 promotion warps arrive
    uint64_t* stg_empty = stg_full + 2;   // [2]: the store warp of that half arrives
    uint64_t* fixbar = stg_empty + 2;     // [2]: split fixup bulk loads, per column half
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(fixbar + 2);
    // MoE: the group offsets in shared memory -- every role's tile cursor walks them at every
    // tile, and from global memory each step of that walk is a dependent L2 round trip
    __shared__ int32_t s_offs[kSmemGroups + 1];
    const bool offs_smem = p.offsets != nullptr && p.groups <= kSmemGroups;
    if (offs_smem)
        for (int i = threadIdx.x; i <= p.groups; i += blockDim.x) s_offs[i] = p.offsets[i];
    const int32_t* offs = offs_smem ? s_offs : nullptr;

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < NBUF; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], NUM_EPI_WARPS);
        }
        for (int hh = 0; hh < 2; ++hh) {
            mbar_init(&stg_full[hh], 4);
            mbar_init(&stg_empty[hh], 1);
            mbar_init(&fixbar[hh], 1);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    if (warp < EPI_WARP0) regs_dec<REGS_CTRL>();

    if (warp == 0) {
        if (lane == 0) {
            // ------------------------------------------------------------ TMA producer
            tma_prefetch_desc(&tmA);
            tma_prefetch_desc(&tmB);
            TileCursor<BM, RASTER_GM> cur;
            cur.init(p, offs);
            uint32_t it = 0;
            int mt, nt;
            // whole tiles, then split slices (work_item); one body instance per form keeps the
            // whole-tile loop's k range in the constant bank (72 registers here)
            auto load_tile = [&](int kb0, int kb1) {
                const int32_t arow = static_cast<int32_t>(cur.row0 + int64_t(mt) * BM);
                const int32_t brow = nt * BN;
                for (int kb = kb0; kb < kb1; ++kb, ++it) {
                    const uint32_t stage = it % STAGES;
                    const uint32_t ph = (it / STAGES) & 1u;
                    mbar_wait(&empty[stage], ph ^ 1u);
                    mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
                    tma_load_2d(smA + stage * A_TILE, &tmA, &full[stage], kb * BK, arow);
                    tma_load_3d(smB + stage * C::B_TILE, &tmB, &full[stage], kb * BK, brow, cur.g);
                }
            };
            int v = blockIdx.x;
            for (; v < p.dp_tiles && cur.seek(p, v, mt, nt); v += gridDim.x) load_tile(0, p.num_kb);
            int sp, kb0, kb1;
            for (; cur.seek(p, work_item(p, v, sp, kb0, kb1), mt, nt); v += gridDim.x) load_tile(kb0, kb1);
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ------------------------------------------------------------ MMA issuer
            const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(tmem_slot);
            TileCursor<BM, RASTER_GM> cur;
            cur.init(p, offs);
            uint32_t it = 0;
            int mt, nt;
            auto mma_tile = [&](int kb0, int kb1) {
                for (int kb = kb0; kb < kb1; ++kb, ++it) {
                    const uint32_t stage = it % STAGES;
                    const uint32_t ph = (it / STAGES) & 1u;
                    const uint32_t buf = it % NBUF;
                    const uint32_t bph = (it / NBUF) & 1u;
                    mbar_wait(&tempty[buf], bph ^ 1u);  // promotion warps drained this buffer
                    mbar_wait(&full[stage], ph);        // TMA landed A and B
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(smA + stage * A_TILE);
                    const uint32_t b0 = smem_u32(smB + stage * C::B_TILE);
                    const uint32_t d = tmem + buf * BN;
#pragma unroll
                    for (int kk = 0; kk < BK / 32; ++kk)
                        mma_f8f6f4(d, smem_desc_k_sw128(a0 + kk * 32), smem_desc_k_sw128(b0 + kk * 32),
                                   C::IDESC, kk > 0 ? 1u : 0u);
                    mma_commit(&empty[stage]);
                    mma_commit(&tfull[buf]);
                }
            };
            int v = blockIdx.x;
            for (; v < p.dp_tiles && cur.seek(p, v, mt, nt); v += gridDim.x) mma_tile(0, p.num_kb);
            int sp, kb0, kb1;
            for (; cur.seek(p, work_item(p, v, sp, kb0, kb1), mt, nt); v += gridDim.x) mma_tile(kb0, kb1);
        }
    } else if ((warp == 2 || warp == 3) && !p.out_f32 && EPI_COLS == 128) {
        // ------------------------------------------------------------ store warps (BF16)
        // (whole tiles only; split tiles are stored by the promotion warps)
        const int h = warp - 2;
        TileCursor<BM, RASTER_GM> cur;
        cur.init(p, offs);
        uint32_t tile_no = 0;
        int mt, nt;
        for (int t = blockIdx.x; t < p.dp_tiles && cur.seek(p, t, mt, nt); t += gridDim.x) {
            const int64_t col0 = int64_t(nt) * BN + h * EPI_COLS;
            if (col0 >= p.n) {  // the promotion warps skip such halves too
                continue;
            }
            store_tile_half(p, smEpi, h, lane, cur.row0 + int64_t(mt) * BM, int64_t(cur.row0) + cur.rows, col0,
                            stg_full, stg_empty, tile_no);
        }
    } else if (warp >= EPI_WARP0) {
        // ---------------------------------------------------------------- promotion warps
        regs_inc<REGS_EPI>();
        const int h = (warp - EPI_WARP0) >> 2;  // column half of the tile
        const int qd = warp & 3;                // TMEM lane quarter this warp may access
        const int r_in_tile = qd * 32 + lane;
        uint8_t* stg = smEpi + (warp - EPI_WARP0) * EPI_CHUNKS * EPI_CHUNK_BYTES;
        if (lane == 0) tma_prefetch_desc(&tmD);
        const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(tmem_slot);
        TileCursor<BM, RASTER_GM> cur;
        cur.init(p, offs);
        uint32_t it = 0;
        uint32_t tile_no = 0;
        int sp = 0, kb0 = 0, kb1 = 0;
        auto make_tile = [&](int tq, int mt, int nt) {
            const bool split = tq >= p.dp_tiles;
            return EpiTile{cur.row0 + int64_t(mt) * BM + r_in_tile, int64_t(cur.row0) + cur.rows,
                           int64_t(nt) * BN + h * EPI_COLS, cur.g, kb0, kb1, split ? tq - p.dp_tiles : 0, sp,
                           split ? p.splits : 1};
        };
        int mt = 0, nt = 0;
        int t = blockIdx.x;  // work item (work_item)
        int tq = work_item(p, t, sp, kb0, kb1);
        bool have = cur.seek(p, tq, mt, nt);
        EpiTile tile = have ? make_tile(tq, mt, nt) : EpiTile{0, 0, 0, 0, 0, 0, 0, 0, 1};
        ScalePre pre = prefetch_scales(p, tile);
        while (have) {
            const int tn = t + gridDim.x;
            tq = work_item(p, tn, sp, kb0, kb1);
            const bool have_next = cur.seek(p, tq, mt, nt);
            const EpiTile next = have_next ? make_tile(tq, mt, nt) : tile;
            ScalePre next_pre = pre;
            promote_tile<BN, NBUF, false>(p, &tmD, stg, smem, fixbar, tile, pre, have_next, next, next_pre, tmem, qd, h,
                                          lane, tfull, tempty, it, stg_full, stg_empty, tile_no);
            tile = next;
            pre = next_pre;
            t = tn;
            have = have_next;
        }
        if (lane == 0) bulk_wait_group<0>();
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(*reinterpret_cast<volatile uint32_t*>(tmem_slot), TMEM_COLS);
    }
}

// ------------------------------------------------------------------------------ CTA pair
// cta_group::2: a cluster of 2 CTAs on 2 SMs computes a 256 x 256 output tile.  CTA r loads A
// rows [m0 + 128r, +128) and B rows [n0 + 128r, +128) into its own smem; the leader's single
// MMA thread issues M=256, N=256 tcgen05.mma that reads A from each CTA's smem for that CTA's
// rows and B from both CTAs' smem, and writes each CTA's 128 rows x 256 fp32 into that CTA's
// TMEM.  Per SM and k-block this moves 32 KB from L2 instead of 48 KB (1-CTA 128x256), the
// operand-traffic ceiling that limited the 1-CTA kernel.  Barriers: full[s] lives in the
// leader (both CTAs' TMA bytes + the peer's arrival land there); empty[s] and tfull[b] are
// arrived in both CTAs by a multicast tcgen05.commit; tempty[b] lives in the leader and
// collects the 16 promotion warps of the pair.
// (Round 1 also measured a 256 x 128 pair tile with four TMEM buffers and a 256 x 256 tile
// committed per 128-column half: both slower -- an N = 128 pair MMA takes as long as N = 256 --
// and removed in round 2.)
template <int PBN>
struct PairCfg {
    static constexpr int BN = PBN;          // tile columns
    static constexpr int B_HALF = PBN / 2;  // B rows loaded by each CTA
    static constexpr int STAGE_BYTES = A_TILE + B_HALF * BK;  // per CTA
    static constexpr int STAGES = SMEM_BUDGET / STAGE_BYTES;
    static constexpr int NBUF = TMEM_COLS / PBN;
    static constexpr uint32_t IDESC = idesc_e4m3_f32(2 * BM, PBN);
    static constexpr size_t SMEM_BYTES = 1024 + size_t(STAGES) * STAGE_BYTES + EPI_STAGE_BYTES + 512;
};
constexpr int PAIR_RASTER_GM = 8;  // pair m-tiles (256 rows) per raster band

template <int PBN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    fp8_block_gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA,
                               const __grid_constant__ CUtensorMap tmB,
                               const __grid_constant__ CUtensorMap tmD, const KParams p) {
    using PC = PairCfg<PBN>;
    constexpr int STAGES = PC::STAGES;
    constexpr int NBUF = PC::NBUF;
    constexpr int PAIR_BN = PC::BN;
    constexpr int PAIR_B_HALF = PC::B_HALF;
    constexpr int PAIR_STAGE_BYTES = PC::STAGE_BYTES;
    constexpr uint32_t PAIR_IDESC = PC::IDESC;
    constexpr int EPI_COLS = PAIR_BN / 2;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint8_t* smA = smem;
    uint8_t* smB = smem + STAGES * A_TILE;
    uint8_t* smEpi = smem + STAGES * PAIR_STAGE_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(smEpi + EPI_STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + NBUF;
    uint64_t* stg_full = tempty + NBUF;
    uint64_t* stg_empty = stg_full + 2;
    uint64_t* fixbar = stg_empty + 2;     // [2]: split fixup bulk loads, per column half
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(fixbar + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int64_t pair = blockIdx.x >> 1;
    const int64_t npairs = gridDim.x >> 1;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 2);   // leader: own arrive.expect_tx + the peer's arrive
            mbar_init(&empty[s], 1);  // multicast commit
        }
        for (int b = 0; b < NBUF; ++b) {
            mbar_init(&tfull[b], 1);                  // multicast commit
            // leader: the promotion warps of both CTAs.  (Funnelling the peer's 8 releases
            // through one forwarded remote arrive was measured: no change.)
            mbar_init(&tempty[b], 2 * NUM_EPI_WARPS);
        }
        for (int hh = 0; hh < 2; ++hh) {
            mbar_init(&stg_full[hh], 4);
            mbar_init(&stg_empty[hh], 1);
            mbar_init(&fixbar[hh], 1);
        }
        fence_mbar_init();
    }
    cluster_sync_all();
    if (warp == 1) tmem_alloc_pair(tmem_slot, TMEM_COLS);
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();

    if (warp < EPI_WARP0) regs_dec<REGS_CTRL>();

    if (warp == 0) {
        if (lane == 0) {
            // ------------------------------------------------------------ TMA producer (both CTAs)
            tma_prefetch_desc(&tmA);
            tma_prefetch_desc(&tmB);
            TileCursor<2 * BM, PAIR_RASTER_GM> cur;
            cur.init(p);
            uint32_t it = 0;
            int mt, nt;
            // whole tiles, then at most one tail-wave slice (pair_item); one body instance per
            // form keeps the whole-tile loop's k range in the constant bank (72 registers here)
            auto load_tile = [&](int kb0, int kb1) {
                const int32_t arow = static_cast<int32_t>(cur.row0 + int64_t(mt) * 2 * BM + rank * BM);
                const int32_t brow = nt * PAIR_BN + static_cast<int32_t>(rank) * PAIR_B_HALF;
                for (int kb = kb0; kb < kb1; ++kb, ++it) {
                    const uint32_t stage = it % STAGES;
                    const uint32_t ph = (it / STAGES) & 1u;
                    mbar_wait(&empty[stage], ph ^ 1u);
                    if (leader)
                        mbar_arrive_expect_tx(&full[stage], 2 * PAIR_STAGE_BYTES);
                    else
                        mbar_arrive_cluster(&full[stage], 0);
                    tma_load_2d_pair(smA + stage * A_TILE, &tmA, &full[stage], kb * BK, arow);
                    tma_load_3d_pair(smB + stage * (PAIR_B_HALF * BK), &tmB, &full[stage], kb * BK, brow, cur.g);
                }
            };
            int v = static_cast<int>(pair);
            for (; v < p.dp_tiles && cur.seek(p, v, mt, nt); v += static_cast<int>(npairs)) load_tile(0, p.num_kb);
            int sp, kb0, kb1;
            for (; cur.seek(p, work_item(p, v, sp, kb0, kb1), mt, nt); v += static_cast<int>(npairs))
                load_tile(kb0, kb1);
        }
    } else if (warp == 1) {
        if (lane == 0 && leader) {
            // ------------------------------------------------------------ MMA issuer (leader)
            const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(tmem_slot);
            TileCursor<2 * BM, PAIR_RASTER_GM> cur;
            cur.init(p);
            uint32_t it = 0;
            int mt, nt;
            auto mma_tile = [&](int kb0, int kb1) {
                for (int kb = kb0; kb < kb1; ++kb, ++it) {
                    const uint32_t stage = it % STAGES;
                    const uint32_t ph = (it / STAGES) & 1u;
                    const uint32_t buf = it % NBUF;
                    const uint32_t bph = (it / NBUF) & 1u;
                    mbar_wait(&tempty[buf], bph ^ 1u);  // both CTAs' promotion warps drained it
                    mbar_wait(&full[stage], ph);        // both CTAs' TMA bytes landed
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(smA + stage * A_TILE);
                    const uint32_t b0 = smem_u32(smB + stage * (PAIR_B_HALF * BK));
                    const uint32_t d = tmem + buf * PAIR_BN;
#pragma unroll
                    for (int kk = 0; kk < BK / 32; ++kk)
                        mma_f8f6f4_pair(d, smem_desc_k_sw128(a0 + kk * 32), smem_desc_k_sw128(b0 + kk * 32),
                                        PAIR_IDESC, kk > 0 ? 1u : 0u);
                    mma_commit_pair(&empty[stage], 0x3);
                    mma_commit_pair(&tfull[buf], 0x3);
                }
            };
            int v = static_cast<int>(pair);
            for (; v < p.dp_tiles && cur.seek(p, v, mt, nt); v += static_cast<int>(npairs)) mma_tile(0, p.num_kb);
            int sp, kb0, kb1;
            for (; cur.seek(p, work_item(p, v, sp, kb0, kb1), mt, nt); v += static_cast<int>(npairs))
                mma_tile(kb0, kb1);
            // the peer's last remote arrivals must land before the barriers go away
            for (uint32_t j = 0; j < NBUF && j < it; ++j) {
                const uint32_t i = it - 1 - j;
                mbar_wait(&tempty[i % NBUF], (i / NBUF) & 1u);
            }
        }
    } else if ((warp == 2 || warp == 3) && !p.out_f32 && EPI_COLS == 128) {
        // ------------------------------------------------------------ store warps (BF16)
        // (only where promote_tile parks BF16 slices for them: 128 columns per half, whole
        // tiles; the split tail tiles are stored by the promotion warps)
        const int h = warp - 2;
        TileCursor<2 * BM, PAIR_RASTER_GM> cur;
        cur.init(p);
        uint32_t tile_no = 0;
        int mt, nt;
        for (int t = static_cast<int>(pair); t < p.dp_tiles && cur.seek(p, t, mt, nt);
             t += static_cast<int>(npairs)) {
            const int64_t col0 = int64_t(nt) * PAIR_BN + h * EPI_COLS;
            if (col0 >= p.n) continue;
            store_tile_half(p, smEpi, h, lane, cur.row0 + int64_t(mt) * 2 * BM + int64_t(rank) * BM,
                            int64_t(cur.row0) + cur.rows, col0, stg_full, stg_empty, tile_no);
        }
    } else if (warp >= EPI_WARP0) {
        // ---------------------------------------------------------------- promotion warps
        regs_inc<REGS_EPI>();
        const int h = (warp - EPI_WARP0) >> 2;
        const int qd = warp & 3;
        const int r_in_tile = qd * 32 + lane;
        uint8_t* stg = smEpi + (warp - EPI_WARP0) * EPI_CHUNKS * EPI_CHUNK_BYTES;
        if (lane == 0) tma_prefetch_desc(&tmD);
        const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(tmem_slot);
        TileCursor<2 * BM, PAIR_RASTER_GM> cur;
        cur.init(p);
        uint32_t it = 0;
        uint32_t tile_no = 0;
        int sp = 0, kb0 = 0, kb1 = 0;
        auto make_tile = [&](int tq, int mt, int nt) {
            const bool split = tq >= p.dp_tiles;
            return EpiTile{cur.row0 + int64_t(mt) * 2 * BM + int64_t(rank) * BM + r_in_tile,
                           int64_t(cur.row0) + cur.rows, int64_t(nt) * PAIR_BN + h * EPI_COLS, cur.g, kb0, kb1,
                           split ? (tq - p.dp_tiles) * 2 + static_cast<int>(rank) : 0, sp, split ? p.splits : 1};
        };
        int mt = 0, nt = 0;
        int t = static_cast<int>(pair);  // work item (pair_item)
        int tq = work_item(p, t, sp, kb0, kb1);
        bool have = cur.seek(p, tq, mt, nt);
        EpiTile tile = have ? make_tile(tq, mt, nt) : EpiTile{0, 0, 0, 0, 0, 0, 0, 0, 1};
        ScalePre pre = prefetch_scales(p, tile);
        while (have) {
            const int tn = t + static_cast<int>(npairs);
            tq = work_item(p, tn, sp, kb0, kb1);
            const bool have_next = cur.seek(p, tq, mt, nt);
            const EpiTile next = have_next ? make_tile(tq, mt, nt) : tile;
            ScalePre next_pre = pre;
            promote_tile<PAIR_BN, NBUF, true>(p, &tmD, stg, smem, fixbar, tile, pre, have_next, next, next_pre, tmem, qd,
                                              h, lane, tfull, tempty, it, stg_full, stg_empty, tile_no);
            tile = next;
            pre = next_pre;
            t = tn;
            have = have_next;
        }
        if (lane == 0) bulk_wait_group<0>();
    }

    tc_fence_before();
    cluster_sync_all();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_pair(*reinterpret_cast<volatile uint32_t*>(tmem_slot), TMEM_COLS);
    }
}

// ------------------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    });
    return fn;
}


struct DeviceInfo {
    int sms = 0;
    bool attr_set = false;
};
DeviceInfo g_dev[64];
std::mutex g_dev_mu;

cudaError_t device_info(int& sms) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lk(g_dev_mu);
    DeviceInfo& di = g_dev[dev];
    if (!di.attr_set) {
        e = cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, dev);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(fp8_block_gemm_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(Cfg<256>::SMEM_BYTES));
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(fp8_block_gemm_pair_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(PairCfg<256>::SMEM_BYTES));
        if (e != cudaSuccess) return e;
        di.attr_set = true;
    }
    sms = di.sms;
    return cudaSuccess;
}

// Split-K plans (BN = 256 tiles).  Work items: whole tiles [0, dp_tiles), then `splits` K slices
// of each of the remaining split_tiles tiles (work_item); a split tile's slices park fp32
// partials in the workspace and the last slice to arrive sums them in slice order
// (deterministic).  Two forms:
//  * decode (one-CTA kernel, M <= 16): every tile split, S minimising the busiest CTA's share
//    ceil(tiles * S / sms) / S of one tile's k-loop (ties to fewer slices), when the tiles fill
//    at most half the SMs;
//  * tail wave (CTA pair, M >= 1024): T tiles on U units (CTA pairs) run in
//    ceil(T / U) waves, the last R = T mod U tiles wide (pair: qkv at M = 8192 768 = 10 x 74 + 28;
//    a P = 8 qkv shard 96 = 74 + 22; a 30B o_proj shard 32 < 74).  The first T - R tiles stay
//    whole, the last R are cut into S = min(U / R, num_kb / 16, 8) slices, so the tail takes
//    1/S of a tile's k-loop instead of one.  Dev A/B: FP8Q_TAIL_SPLIT=0.
struct SplitPlan {
    int splits = 1;
    int dp_tiles = 0x7fffffff;
    int64_t split_tiles = 0;
    int ctas = 1;  // CTAs per tile (2: CTA pair, each parks its own 128 rows)
    bool bulk = false;  // every CTA (pair) gets at most one slice, as its last work item
};
SplitPlan plan_split(int64_t m, int64_t n, int64_t k, int sms, bool pair) {
    static const bool tail_enabled = [] {
        const char* e = std::getenv("FP8Q_TAIL_SPLIT");
        return !(e != nullptr && e[0] == '0');
    }();
    SplitPlan sp;
    sp.ctas = pair ? 2 : 1;
    const int64_t tile_rows = pair ? 2 * BM : BM;
    const int64_t tiles = ((m + tile_rows - 1) / tile_rows) * ((n + 255) / 256);
    const int64_t units = pair ? sms / 2 : sms;
    const int64_t num_kb = k / BK;
    if (tiles <= 0 || units <= 0 || m <= 0) return sp;
    if (!pair && m <= 16) {
        // measured (tools/kernel_bench.py --decode): the all-tiles split pays only for the
        // smallest M, where the parked fp32 partials are tiny
        if (tiles * 2 > sms || num_kb < 2) return sp;
        int best = 1;
        double best_cost = 1e30;
        for (int s = 1; s <= 16 && 2 * s <= num_kb; ++s) {
            const double cost = static_cast<double>((tiles * s + sms - 1) / sms) / s;
            if (cost < best_cost - 1e-9) {
                best_cost = cost;
                best = s;
            }
        }
        if (best > 1) {
            sp.splits = best;
            sp.dp_tiles = 0;
            sp.split_tiles = tiles;
        }
        return sp;
    }
    // measured (tools/one_shape.py, graph timings, split vs FP8Q_TAIL_SPLIT=0, two boxes): the
    // fixup costs a few microseconds (park 128 KB per CTA, the last slice bulk-reads S x 128 KB),
    // so it pays on the CTA pair with long slices and many m-tiles -- at M = 8192 N = 768 / 256
    // / 1536 (K = 4096) 37.5 -> 36.4 / 21.8 -> 20.7 / 56.9 -> 53.0 us, (2048, 512, 4096) 22.1 ->
    // 19.7, down_proj P = 2 shard (8192, 2048, 12288) 201.7 -> 187.4 -- and loses with
    // 5-8 k-block slices (K = 2048: (8192, 640, 2048) 27.1 -> 30.0, (8192, 1280, 2048) 31.6 ->
    // 33.4), at M = 256 (gate_up 38.3 -> 39.6) and on the one-CTA kernel ((200, 24576, 2048):
    // 24.6 -> 26.3); those stay unsplit.
    if (!tail_enabled || !pair || m < 2 * BM) return sp;
    const int64_t r = tiles % units;
    if (r == 0) return sp;
    // one slice per unit at most (R S <= U), so every slice is its CTA's last item and the
    // fixup can use the idle shared-memory ring; >= 16 k-blocks per slice
    const int64_t s = std::min<int64_t>(std::min<int64_t>(units / r, num_kb / 16), 8);
    if (s < 2) return sp;
    // below M = 1024 only without a whole wave and with the slices on >= 64 % of the SMs: then
    // the split pair beats the swap-AB cluster kernel at decode M = 256 (measured, one box:
    // down_proj 31.0 -> 27.7 us on 128 SMs, qkv 23.9 -> 21.0 on 96; o_proj, 64 SMs, 16.9 ->
    // 20.6 stays on the cluster kernel; gate_up, one whole wave + 22 tiles, 38.3 -> 38.4)
    if (m < 8 * BM && !(tiles < units && 100 * (2 * r * s) >= 64 * sms)) return sp;
    sp.bulk = true;
    sp.splits = static_cast<int>(s);
    sp.dp_tiles = static_cast<int>(tiles - r);
    sp.split_tiles = r;
    return sp;
}
// Workspace: [counters: SPLIT_COUNTER_BYTES][partials [split tile][slice][cta][128][256] fp32];
// the counter region sits at a fixed offset so the "left zeroed" invariant holds whatever shape
// used the workspace before.
constexpr size_t SPLIT_COUNTER_BYTES = 4096;  // >= 4 B x split_tiles x ctas (<= sms)
size_t split_ws_bytes(const SplitPlan& sp) {
    if (sp.splits <= 1) return 0;
    return SPLIT_COUNTER_BYTES + static_cast<size_t>(sp.split_tiles * sp.splits * sp.ctas * BM * 256) * 4;
}

// Kernel choice (see launch_cfg): env FP8Q_GEMM_KIND = 256 | 1256 overrides (dev only).
// Default: the CTA-pair kernel for dense M >= 256, the one-CTA 128 x 256 kernel otherwise.
int choose_kind(const GemmArgs& a) {
    static int forced = [] {
        const char* e = std::getenv("FP8Q_GEMM_KIND");
        return e ? std::atoi(e) : 0;
    }();
    if (forced == 256 || forced == 1256) return forced;
    // Measured (tools/kernel_bench.py --moe, Qwen3-30B-A3B experts): the grouped GEMM's short
    // per-expert k-loops (fc2: 6 k-blocks) and ragged segments favour the one-CTA 128 x 256
    // tile (+5 % at T = 8192, +34-41 % at T = 1024) over the CTA pair.
    if (a.offsets != nullptr) return 256;
    if (a.m < 2 * BM) return 256;
    return 1256;
}

// kind: 256 = one-CTA kernel, 128 x 256 tiles; 1256 = CTA-pair kernel, 256 x 256 tiles.
template <int KIND>
cudaError_t launch_cfg(const GemmArgs& a, PFN_cuTensorMapEncodeTiled_v12000 encode, int sms,
                       cudaStream_t stream) {
    constexpr bool kPair = KIND > 1000;
    constexpr int BN = kPair ? KIND - 1000 : KIND;
    constexpr int B_BOX = kPair ? BN / 2 : KIND;
    CUtensorMap tmA, tmB;
    {
        cuuint64_t dims[2] = {static_cast<cuuint64_t>(a.k), static_cast<cuuint64_t>(a.m)};
        cuuint64_t strides[1] = {static_cast<cuuint64_t>(a.ld_a)};
        cuuint32_t box[2] = {BK, BM};
        cuuint32_t estr[2] = {1, 1};
        CUresult r = encode(&tmA, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(a.a), dims,
                            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    }
    {
        const int64_t g = a.offsets != nullptr ? a.groups : 1;
        const int64_t sb = (g > 1) ? a.stride_b : a.ld_b * a.n;
        cuuint64_t dims[3] = {static_cast<cuuint64_t>(a.k), static_cast<cuuint64_t>(a.n),
                              static_cast<cuuint64_t>(g)};
        cuuint64_t strides[2] = {static_cast<cuuint64_t>(a.ld_b), static_cast<cuuint64_t>(sb)};
        cuuint32_t box[3] = {BK, static_cast<cuuint32_t>(B_BOX), 1};
        cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = encode(&tmB, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(a.b), dims,
                            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    }
    CUtensorMap tmD;
    {
        const int esz = a.out_f32 ? 4 : 2;
        cuuint64_t dims[2] = {static_cast<cuuint64_t>(a.n), static_cast<cuuint64_t>(a.m)};
        cuuint64_t strides[1] = {static_cast<cuuint64_t>(a.ld_d * esz)};
        cuuint32_t box[2] = {static_cast<cuuint32_t>(64 / esz), 32};
        cuuint32_t estr[2] = {1, 1};
        CUresult r = encode(&tmD, a.out_f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                            2, a.d, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    }
    KParams p;
    p.sa = a.sa;
    p.ld_sa = a.ld_sa;
    p.sb = a.sb;
    p.ld_sb = a.ld_sb;
    p.stride_sb = a.stride_sb;
    p.d = a.d;
    p.ld_d = a.ld_d;
    p.out_f32 = a.out_f32 ? 1 : 0;
    p.m = a.m;
    p.n = a.n;
    p.num_kb = static_cast<int>(a.k / BK);
    p.num_n_tiles = static_cast<int>((a.n + BN - 1) / BN);
    p.offsets = a.offsets;
    p.groups = a.offsets != nullptr ? a.groups : 1;
    p.splits = 1;
    p.ws = nullptr;
    p.counters = nullptr;
    p.dp_tiles = 0x7fffffff;
    p.fix_bulk = 0;
    {
        // raster band: as many m-tiles as keep the band's A panel (rows x K bytes) within
        // ~32 MB of L2, so B streams from HBM once per band (FP8Q_GEMM_RASTER overrides, dev)
        static const int forced_raster = [] {
            const char* e = std::getenv("FP8Q_GEMM_RASTER");
            return e ? std::atoi(e) : 0;
        }();
        const int64_t tile_rows = kPair ? 2 * BM : BM;
        int64_t r = (32LL << 20) / (tile_rows * (a.k > 0 ? a.k : 1));
        r = r < 4 ? 4 : (r > 64 ? 64 : r);
        // measured (FP8Q_GEMM_RASTER sweep, pair kernel): gate_up (K = 4096) +1.5 % at 32
        // m-tiles per band vs 8; down (K = 12288) best at 8-16; qkv / o insensitive
        p.raster = forced_raster != 0 ? forced_raster : (kPair ? static_cast<int>(r) : RASTER_GM);
        // B smaller than A and all of it fits in ~64 MB of L2 (down_proj: B 50 MB vs A 100 MB):
        // keep B resident instead -- bands of n-tiles covering all of N, n fastest, so A streams
        // from HBM once and B once (the m-band raster re-reads B once per band: 2.8x the operand
        // bytes for down_proj)
        static const bool b_resident = [] {  // dev A/B: FP8Q_GEMM_BRES=0 keeps the m-band raster
            const char* e = std::getenv("FP8Q_GEMM_BRES");
            return !(e != nullptr && e[0] == '0');
        }();
        if (forced_raster == 0 && kPair && b_resident && a.offsets == nullptr && a.n < a.m &&
            a.n * a.k <= (64LL << 20))
            p.raster = -p.num_n_tiles;
    }
    // work items (whole tiles, then split slices) of a dense problem
    int64_t items = ((a.m + (kPair ? 2 * BM : BM) - 1) / (kPair ? 2 * BM : BM)) * p.num_n_tiles;
    if (BN == 256 && a.offsets == nullptr) {
        const SplitPlan sp = plan_split(a.m, a.n, a.k, sms, kPair);
        const size_t need = split_ws_bytes(sp);
        if (sp.splits > 1 && a.workspace != nullptr && a.workspace_bytes >= need) {
            p.splits = sp.splits;
            p.dp_tiles = sp.dp_tiles;
            p.counters = static_cast<int32_t*>(a.workspace);
            p.ws = reinterpret_cast<float*>(static_cast<char*>(a.workspace) + SPLIT_COUNTER_BYTES);
            items = sp.dp_tiles + sp.split_tiles * sp.splits;
            p.fix_bulk = sp.bulk ? 1 : 0;
        }
    }

    if (kPair) {
        int64_t clusters = sms / 2;
        if (a.offsets == nullptr) clusters = items < clusters ? items : clusters;
        fp8_block_gemm_pair_kernel<BN><<<static_cast<unsigned>(2 * clusters), NUM_THREADS, PairCfg<BN>::SMEM_BYTES,
                                         stream>>>(tmA, tmB, tmD, p);
    } else {
        int64_t grid = sms;
        if (a.offsets == nullptr) grid = items < sms ? items : sms;
        fp8_block_gemm_kernel<BN><<<static_cast<unsigned>(grid), NUM_THREADS, Cfg<BN>::SMEM_BYTES, stream>>>(
            tmA, tmB, tmD, p);
    }
    return cudaGetLastError();
}

}  // namespace

void* tensor_map_encode_fn() { return reinterpret_cast<void*>(tensor_map_encoder()); }

bool pair_tail_split_applies(int64_t m, int64_t n, int64_t k, size_t workspace_bytes) {
    int sms = 0;
    if (m < 2 * BM || device_info(sms) != cudaSuccess) return false;
    const SplitPlan sp = plan_split(m, n, k, sms, true);
    return sp.splits > 1 && workspace_bytes >= split_ws_bytes(sp);
}

size_t gemm_workspace_bytes(int64_t m, int64_t n, int64_t k, bool grouped) {
    if (grouped || m <= 0 || n <= 0 || k <= 0) return 0;
    int sms = 0;
    if (device_info(sms) != cudaSuccess) sms = 148;
    // the kernel choose_kind makes by default: the CTA pair from M = 256
    size_t need = split_ws_bytes(plan_split(m, n, k, sms, m >= 2 * BM));
    if (m <= kSkinnyMaxM) need = std::max(need, skinny_workspace_bytes(m, n, k));
    return need;
}

cudaError_t launch_fp8_block_gemm(const GemmArgs& a, cudaStream_t stream, int* launches) {
    *launches = 0;
    if (a.m == 0 || a.n == 0 || a.groups == 0) return cudaSuccess;
    auto encode = tensor_map_encoder();
    if (encode == nullptr) return cudaErrorNotSupported;
    if (skinny_gemm_applies(a)) {
        const cudaError_t es = launch_fp8_gemm_skinny(a, reinterpret_cast<void*>(encode), stream);
        if (es == cudaSuccess) *launches = 1;
        return es;
    }
    int sms = 0;
    cudaError_t e = device_info(sms);
    if (e != cudaSuccess) return e;
    switch (choose_kind(a)) {
        case 256: e = launch_cfg<256>(a, encode, sms, stream); break;
        default: e = launch_cfg<1256>(a, encode, sms, stream); break;
    }
    if (e == cudaSuccess) *launches = 1;
    return e;
}

}  // namespace fp8q
