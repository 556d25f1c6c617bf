// gemm_skinny.cu -- blockwise-scaled FP8 GEMM for decode-sized M (M <= 128).
//
// Same result as gemm.cu:
//     D[m,n] = sum_kb (sa[kb][m] * sb[n/128][kb]) * P_kb[m,n]
// but with the operands swapped so the tiny token count sits in the MMA's N dimension:
//     D^T tile [128 weight rows x MT tokens] = W_tile[128 x K] * X[MT x K]^T
// At M <= 128 the problem is a weight stream (arithmetic intensity <= 2M flop per weight byte,
// below the FP8/HBM ridge), so what matters is keeping every SM's TMA queue full of weight
// tiles.  The work is the sequence of (128-row weight tile = one scale n-block, k-block)
// pairs, T = tiles * k/128 of them, cut into G equal contiguous ranges, one per CTA of a
// persistent grid (stream-K): every SM streams the same number of weight bytes (+-1 k-block)
// whatever the tile count, and the ring holds 6-11 k-blocks of weights in flight per SM.  A
// range is walked as segments (its part of each tile); a tile covered by several CTAs is
// finished by a deterministic fixup (below).
// When whole tiles would leave at least half the SMs idle (qkv, o_proj, down_proj: 32-48
// tiles), the kernel instead runs as CLUSTER split-K: a cluster of cs <= 8 CTAs per weight
// tile, CTA rank r streaming k-blocks [r KB/cs, (r+1) KB/cs); each CTA parks its fp32 partial
// in its own (by then idle) weight ring and, after one cluster barrier, sums a 1/cs slice of
// the tile over the cluster's CTAs in rank order through distributed shared memory.  The
// per-CTA timeline showed the stream-K fixup (fence, counter atomics, one dependent L2 round
// trip per contributor, 64 KB of partials per contributor at M = 128) ending 5-12 us after the
// last weight byte arrived; the DSMEM reduction replaces it with two cluster barriers.
// When every range spans at least one tile's k-blocks (>= 148 tiles, e.g. gate_up), a tile has
// at most two CTAs and the stream-K runs ORDERED: each CTA does the head of its last tile first
// (parked + flagged), then its whole tiles, then the tail of its first tile, which it combines
// with the long-published head -- no atomics, and no fixup round trips after the stream.
// One CTA per SM (the full ring at every M): with two per SM, programmatic dependent launch let
// the block scheduler put two CTAs of the SAME grid on one SM (up to 34 of 148 at M = 1), and
// those streamed their ranges 3-4 us late.  The dependants are released after the producer's
// last TMA issue (the tail), not at entry.
//
// CTA = 12 warps (3 warpgroups):
//   warp 0       TMA producer: per k-block W 128x128 B, X MTx128 B (rows >= m zero-filled by
//                the tensor map) and the k-block's MT activation scales (one TMA row of the
//                MN-major scale matrix) into a 6-11-stage ring (128-byte swizzle).
//   warp 1       TMEM owner + MMA issuer: 4 x tcgen05.mma.kind::f8f6f4 (M=128, N=MT, K=32)
//                per k-block into TMEM buffer it % NBUF (fresh accumulation per k-block).
//   warps 2, 3   idle (they only give their registers to the promotion warps).
//   warps 4..11  promotion: warp w reads TMEM lanes 32*(w%4).. (its 32 weight rows) and half
//                of the MT token columns; acc[j] += P_kb[j] * (sa[kb][j] * sb[nb][kb]) (the
//                same fp32 operations, in the same k order, as gemm.cu), scales from the
//                stage (no dependent global load in the k-loop).  A segment that covers a
//                whole tile is stored at once (BF16 = RNE of the fp32 value).  A partial
//                segment (only the first and the last of a CTA's range can be partial) parks
//                its fp32 partial in the workspace without waiting; after its range the CTA
//                fences once and, per parked tile, bumps the tile's counter: the last CTA of
//                the tile to arrive sums every CTA's partial in CTA order (deterministic: the
//                order never depends on which CTA arrives last) and stores the tile.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "group_quant.cuh"
#include "ptx.cuh"
#include "quant_kernels.h"
#include "scale_tables.cuh"
#include "trace.cuh"

namespace fp8q {
namespace {

constexpr int SK_BN = 128;  // weight rows per tile (MMA M) = one scale n-block
constexpr int SK_BK = 128;
constexpr int SK_THREADS = 384;   // warpgroup 0: TMA, MMA, 2 idle; warpgroups 1-2: promotion
constexpr int SK_EPI_WARP0 = 4;
// setmaxnreg: warpgroup 0 drops to 72 registers so the promotion warpgroups can take 216
// (the CTA's pool is fixed at launch: 384 x 168 = 128 x 72 + 256 x 216).
constexpr int SK_REGS_CTRL = 72;
constexpr int SK_REGS_EPI = 216;
static_assert(128 * (168 - SK_REGS_CTRL) >= 256 * (SK_REGS_EPI - 168), "register pool overdrawn");
constexpr int SK_EPI_WARPS = 8;
constexpr int SK_SMEM_BUDGET = 200 * 1024;
constexpr size_t SK_COUNTER_BYTES = 4096;  // one int32 per tile: up to 1024 tiles (N <= 131072)

constexpr int pow2_at_least(int v, int lo) {
    int p = lo;
    while (p < v) p *= 2;
    return p;
}

template <int MT>
struct SkCfg {
    static constexpr int W_TILE = SK_BN * SK_BK;   // 16 KB
    static constexpr int X_TILE = MT * SK_BK;      // MT x 128 B (a multiple of 1024 B: SW128 atoms)
    static constexpr int SA_BYTES = MT * 4;                          // TMA box bytes
    static constexpr int SA_SLOT = SA_BYTES < 128 ? 128 : SA_BYTES;  // TMA smem dst: 128-B aligned
    static constexpr int STAGE_BYTES = W_TILE + X_TILE;
    static constexpr int TX_BYTES = STAGE_BYTES + SA_BYTES;  // TMA bytes per stage
    static constexpr int STAGES_RAW = SK_SMEM_BUDGET / (STAGE_BYTES + SA_SLOT);
    static constexpr int STAGES = STAGES_RAW > 12 ? 12 : STAGES_RAW;
    static constexpr int NBUF_RAW = 512 / MT;
    static constexpr int NBUF = NBUF_RAW > 8 ? 8 : NBUF_RAW;  // TMEM partial buffers
    static constexpr int TMEM_COLS = pow2_at_least(NBUF * MT, 32);
    static constexpr int COLS = MT / 2;  // token columns per promotion thread
    static constexpr uint32_t IDESC = idesc_e4m3_f32(SK_BN, MT);
    static constexpr size_t SMEM_BYTES = 1024 + size_t(STAGES) * (STAGE_BYTES + SA_SLOT) + 512;
    static_assert(MT % 16 == 0 && MT >= 16 && MT <= 256, "MMA N for M=128 must be a multiple of 16, <= 256");
    static_assert(X_TILE % 1024 == 0, "X tile must be whole 128-byte-swizzle atoms");
    // cluster split-K parks its partial in the (contiguous) W and X rings
    static_assert(STAGES * (W_TILE + X_TILE) >= MT * SK_BN * 4, "no room for the cluster split-K partial");
};

// Fused activation quantization (fp8_linear_dynamic at m <= 16, MT = 16): the ring carries only
// weight tiles; the CTA's activation codes live in a persistent region of up to kFxSlots
// k-blocks (16 rows x 128 B each, SW128 layout) with their scales, written once by the
// promotion warps after griddepcontrol.wait (no separate quantizer launch, no global round trip).
constexpr int kFxSlots = 32;
struct SkFxCfg {
    static constexpr int MT = 16;
    static constexpr int W_TILE = SK_BN * SK_BK;
    static constexpr int X_SLOT = MT * SK_BK;  // 2 KB
    static constexpr int STAGES = 8;
    static constexpr size_t SMEM_BYTES =
        1024 + size_t(STAGES) * W_TILE + size_t(kFxSlots) * X_SLOT + kFxSlots * MT * 4 + 512;
    static_assert(STAGES * W_TILE >= MT * SK_BN * 4, "no room for the cluster split-K partial");
};

struct SkParams {
    const float* sb;
    int64_t ld_sb;
    void* d;
    int64_t ld_d;
    int out_f32;
    int m, n, num_kb, tiles;
    int streamk;        // 1: ranges [c*T/G, (c+1)*T/G) per CTA; 0: whole tiles, strided;
                        // 2: cluster split-K -- cluster = one tile, CTA rank r its k-blocks
                        //    [r*KB/cs, (r+1)*KB/cs), partials reduced through DSMEM;
                        // 3: ordered stream-K (ranges >= KB, so a tile has <= 2 CTAs): the
                        //    range's last, partial tile first (parked + flagged), whole tiles,
                        //    then its first, partial tile, combined with the parked head
    int cs;             // cluster size (mode 2)
    int64_t total;      // T = tiles * num_kb
    float* ws;          // stream-K partials: two [MT][128] fp32 slots per CTA
    int32_t* counters;  // [tiles], left zeroed
    int prefetch;       // weight stages issued before griddepcontrol.wait (dev A/B: FP8Q_SKINNY_PREFETCH)
    const uint16_t* x;  // fused activation quantization: BF16 activations [m][ld_x] (else null)
    int64_t ld_x;
    int32_t* flag;      // non-finite flag of the fused quantization (nullable)
};
__device__ __forceinline__ void grid_dependency_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Walks this CTA's segments: (tile, kb0, kb1) = k-blocks [kb0, kb1) of weight tile `tile`.
template <bool kOrdered>  // false: the ordered stream-K branch compiled out (MT = 256, cluster mode only)
struct SegIterT {
    int64_t x, end;  // stream-K: position in [0, T) and this CTA's range end
    int t;           // tiled: next tile (ordered stream-K: next whole tile)
    int phase;       // ordered stream-K: 0 head of the last tile, 1 whole tiles, 2 tail of the first, 3 done
    __device__ __forceinline__ void init(const SkParams& p) {
        if (p.streamk == 1 || p.streamk == 3) {
            x = static_cast<int64_t>(blockIdx.x) * p.total / gridDim.x;
            end = static_cast<int64_t>(blockIdx.x + 1) * p.total / gridDim.x;
        }
        t = blockIdx.x;
        if (kOrdered && p.streamk == 3) {
            t = static_cast<int>((x + p.num_kb - 1) / p.num_kb);  // first whole tile
            phase = 0;
        }
    }
    __device__ __forceinline__ bool next(const SkParams& p, int& tile, int& kb0, int& kb1) {
        if (kOrdered && p.streamk == 3) {
            if (phase == 0) {
                phase = 1;
                if (end % p.num_kb != 0) {  // head of the range's last tile (shared with the next CTA)
                    tile = static_cast<int>(end / p.num_kb);
                    kb0 = 0;
                    kb1 = static_cast<int>(end % p.num_kb);
                    return true;
                }
            }
            if (phase == 1) {
                if (t < static_cast<int>(end / p.num_kb)) {
                    tile = t++;
                    kb0 = 0;
                    kb1 = p.num_kb;
                    return true;
                }
                phase = 2;
            }
            if (phase == 2) {
                phase = 3;
                if (x % p.num_kb != 0) {  // tail of the range's first tile (shared with the previous CTA)
                    tile = static_cast<int>(x / p.num_kb);
                    kb0 = static_cast<int>(x % p.num_kb);
                    kb1 = p.num_kb;
                    return true;
                }
            }
            return false;
        }
        if (p.streamk == 2) {  // one segment: rank r of cluster `tile`
            if (t < 0) return false;
            const int r = static_cast<int>(blockIdx.x) % p.cs;
            tile = static_cast<int>(blockIdx.x) / p.cs;
            kb0 = r * p.num_kb / p.cs;
            kb1 = (r + 1) * p.num_kb / p.cs;
            t = -1;
            return true;
        }
        if (p.streamk == 1) {
            if (x >= end) return false;
            tile = static_cast<int>(x / p.num_kb);
            const int64_t t0 = int64_t(tile) * p.num_kb;
            kb0 = static_cast<int>(x - t0);
            kb1 = static_cast<int>(end - t0 < p.num_kb ? end - t0 : p.num_kb);
            x = t0 + kb1;
            return true;
        }
        if (t >= p.tiles) return false;
        tile = t;
        kb0 = 0;
        kb1 = p.num_kb;
        t += gridDim.x;
        return true;
    }
};
// The CTA whose range holds k-block position x: the largest c with floor(c T / G) <= x.
__device__ __forceinline__ int sk_cta_of(const SkParams& p, int64_t x) {
    return static_cast<int>(((x + 1) * gridDim.x - 1) / p.total);
}

template <int N>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, float (&v)[N]);
template <>
__device__ __forceinline__ void tmem_ld_cols<8>(uint32_t taddr, float (&v)[8]) {
    uint32_t* r = reinterpret_cast<uint32_t*>(v);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                   "=r"(r[7])
                 : "r"(taddr));
}
template <>
__device__ __forceinline__ void tmem_ld_cols<16>(uint32_t taddr, float (&v)[16]) {
    uint32_t* r = reinterpret_cast<uint32_t*>(v);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
// D[j0 + j][n_row] for j < jn (a running pointer: not COLS precomputed 64-bit addresses).
template <int COLS>
__device__ __forceinline__ void sk_store(const SkParams& p, int64_t n_row, int j0, int jn, const float (&acc)[COLS]) {
    if (p.out_f32) {
        float* d = static_cast<float*>(p.d) + n_row + int64_t(j0) * p.ld_d;
#pragma unroll
        for (int j = 0; j < COLS; ++j) {
            if (j < jn) *d = acc[j];
            d += p.ld_d;
        }
    } else {
        __nv_bfloat16* d = static_cast<__nv_bfloat16*>(p.d) + n_row + int64_t(j0) * p.ld_d;
#pragma unroll
        for (int j = 0; j < COLS; ++j) {
            if (j < jn) *d = __float2bfloat16_rn(acc[j]);
            d += p.ld_d;
        }
    }
}

// The CTA's activation k-blocks in the fused mode: [kx0, kx0 + nkx) (the host guarantees
// nkx <= kFxSlots); a range that crosses a tile boundary takes all k-blocks.
__device__ __forceinline__ void sk_fx_range(const SkParams& p, int& kx0, int& nkx) {
    if (p.streamk == 2) {
        const int r = static_cast<int>(cluster_ctarank());
        kx0 = r * p.num_kb / p.cs;
        nkx = (r + 1) * p.num_kb / p.cs - kx0;
    } else if (p.streamk == 1 || p.streamk == 3) {
        const int64_t x = static_cast<int64_t>(blockIdx.x) * p.total / gridDim.x;
        const int64_t e = static_cast<int64_t>(blockIdx.x + 1) * p.total / gridDim.x;
        if (e <= x) {
            kx0 = 0;
            nkx = 0;
        } else if (x / p.num_kb == (e - 1) / p.num_kb) {
            kx0 = static_cast<int>(x % p.num_kb);
            nkx = static_cast<int>(e - x);
        } else {
            kx0 = 0;
            nkx = p.num_kb;
        }
    } else {
        kx0 = 0;
        nkx = p.num_kb;
    }
}

template <int MT, bool kFX = false>
__global__ void __launch_bounds__(SK_THREADS, 1)
    fp8_gemm_skinny_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                           const __grid_constant__ CUtensorMap tmS, const SkParams p) {
    using C = SkCfg<MT>;
    using SegIter = SegIterT<(MT <= 128)>;
    static_assert(!kFX || MT == 16, "fused activation quantization: MT = 16 only");
    constexpr int STAGES = kFX ? SkFxCfg::STAGES : C::STAGES;
    constexpr int NBUF = C::NBUF;
    constexpr int COLS = C::COLS;
    constexpr int SA_STRIDE = C::SA_SLOT / 4;  // floats between stages' scale slots
    constexpr uint32_t TX_BYTES = kFX ? static_cast<uint32_t>(C::W_TILE) : static_cast<uint32_t>(C::TX_BYTES);
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint8_t* smW = smem;
    // kFX: smX = the persistent activation-code region (kFxSlots x 2 KB), smS its scales [slot][16]
    uint8_t* smX = smW + STAGES * C::W_TILE;
    float* smS = reinterpret_cast<float*>(smX + (kFX ? kFxSlots * SkFxCfg::X_SLOT : STAGES * C::X_TILE));
    uint64_t* full = reinterpret_cast<uint64_t*>(smS + (kFX ? kFxSlots * MT : STAGES * SA_STRIDE));
    uint64_t* empty = full + STAGES;    // the MMA consumed W and X of the stage
    uint64_t* sempty = empty + STAGES;  // the promotion warps consumed its activation scales
    uint64_t* tfull = sempty + STAGES;
    uint64_t* tempty = tfull + NBUF;
    uint64_t* xready = tempty + NBUF;   // kFX: the activation codes and scales are in shared memory
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xready + 1);
    __shared__ ScaleTables tabs;
    int kx0 = 0, nkx = 0;
    if (kFX) sk_fx_range(p, kx0, nkx);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t trace_tag = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(p.sb));
    (void)trace_tag;
    if (threadIdx.x == 0) FP8Q_TREC(trace_tag, 0);
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
            mbar_init(&sempty[s], SK_EPI_WARPS);
        }
        for (int b = 0; b < NBUF; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], SK_EPI_WARPS);
        }
        mbar_init(xready, 1);
        fence_mbar_init();
    }
    if (kFX) init_scale_tables(tabs);
    if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp < SK_EPI_WARP0) regs_dec<SK_REGS_CTRL>();

    if (warp == 0) {
        if (lane == 0) {
            // ------------------------------------------------------------ TMA producer
            tma_prefetch_desc(&tmW);
            tma_prefetch_desc(&tmX);
            tma_prefetch_desc(&tmS);
            // Programmatic dependent launch: the weights (and their scales) are never written by
            // the kernel this one may overlap (only this kernel triggers early, see below), so
            // the first ring fill of weight tiles is issued before waiting for the previous
            // grid; the activations and their scales (its possible outputs) only after.
            uint32_t it = 0;
            SegIter seg;
            seg.init(p);
            int tile, kb0, kb1;
            uint32_t npf = 0;  // weight stages already in flight
            {
                SegIter pre = seg;
                int pt, pk0, pk1;
                uint32_t n = 0;
                const uint32_t cap = min(static_cast<uint32_t>(STAGES), static_cast<uint32_t>(p.prefetch));
                while (n < cap && pre.next(p, pt, pk0, pk1))
                    for (int kb = pk0; kb < pk1 && n < cap; ++kb, ++n) {
                        mbar_arrive_expect_tx(&full[n], TX_BYTES);
                        tma_load_2d(smW + n * C::W_TILE, &tmW, &full[n], kb * SK_BK, pt * SK_BN);
                    }
                npf = n;
            }
            grid_dependency_wait();
            FP8Q_TREC(trace_tag, 1);
            while (seg.next(p, tile, kb0, kb1)) {
                for (int kb = kb0; kb < kb1; ++kb, ++it) {
                    const uint32_t stage = it % STAGES;
                    const uint32_t ph = (it / STAGES) & 1u;
                    const bool prefetched = it < npf;  // W already in flight, expect_tx armed
                    if (!prefetched) {
                        mbar_wait(&empty[stage], ph ^ 1u);
                        if (!kFX) mbar_wait(&sempty[stage], ph ^ 1u);
                    }
                    if (!prefetched) {
                        mbar_arrive_expect_tx(&full[stage], TX_BYTES);
                        tma_load_2d(smW + stage * C::W_TILE, &tmW, &full[stage], kb * SK_BK, tile * SK_BN);
                    }
                    if (!kFX) {
                        tma_load_2d(smX + stage * C::X_TILE, &tmX, &full[stage], kb * SK_BK, 0);
                        tma_load_2d(smS + stage * SA_STRIDE, &tmS, &full[stage], 0, kb);
                    }
                }
            }
            FP8Q_TREC(trace_tag, 2);
            // every weight byte is requested: let the next kernel in the stream (programmatic
            // stream serialization) launch and start its prologue / weight prefetch in our tail
            asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ------------------------------------------------------------ MMA issuer
            const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(tmem_slot);
            uint32_t it = 0;
            SegIter seg;
            seg.init(p);
            int tile, kb0, kb1;
            if (kFX) mbar_wait(xready, 0);  // the CTA's activation codes are in shared memory
            while (seg.next(p, tile, kb0, kb1)) {
                for (int kb = kb0; kb < kb1; ++kb, ++it) {
                    const uint32_t stage = it % STAGES;
                    const uint32_t ph = (it / STAGES) & 1u;
                    const uint32_t buf = it % NBUF;
                    const uint32_t bph = (it / NBUF) & 1u;
                    mbar_wait(&tempty[buf], bph ^ 1u);
                    mbar_wait(&full[stage], ph);
                    if (it == 0) FP8Q_TREC(trace_tag, 3);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(smW + stage * C::W_TILE);
                    const uint32_t b0 = kFX ? smem_u32(smX + (kb - kx0) * SkFxCfg::X_SLOT)
                                            : smem_u32(smX + stage * C::X_TILE);
                    const uint32_t d = tmem + buf * MT;
#pragma unroll
                    for (int kk = 0; kk < SK_BK / 32; ++kk)
                        mma_f8f6f4(d, smem_desc_k_sw128(a0 + kk * 32), smem_desc_k_sw128(b0 + kk * 32), C::IDESC,
                                   kk > 0 ? 1u : 0u);
                    mma_commit(&empty[stage]);
                    mma_commit(&tfull[buf]);
                }
            }
            FP8Q_TREC(trace_tag, 4);
        }
    } else if (warp >= SK_EPI_WARP0) {
        // ---------------------------------------------------------------- promotion warps
        regs_inc<SK_REGS_EPI>();
        grid_dependency_wait();  // before any global write (D, workspace): the previous grid is done
        if (kFX) {
            // ---- fused activation quantization (the quantizers' element map, group_quant.cuh):
            // group (token j, k-block kx0 + s) -> 128 codes at row j of slot s (SW128: 16-byte
            // chunk c of row j at chunk position c ^ (j & 7)) and its scale at smS[s][j]; rows
            // m..15 (the MMA's zero padding) get zero codes and scales.  One warp per group: lane
            // l holds channels 4l..4l+3.
            const int ew = warp - SK_EPI_WARP0;
            const int m = p.m;
            for (int i = ew * 32 + lane; i < nkx * (MT - m) * 8; i += SK_EPI_WARPS * 32) {
                const int s = i / ((MT - m) * 8), rem = i - s * (MT - m) * 8;
                const int j = m + rem / 8, c = rem % 8;
                st_shared_v4(smem_u32(smX + s * SkFxCfg::X_SLOT + j * 128 + c * 16), 0u, 0u, 0u, 0u);
            }
            for (int i = ew * 32 + lane; i < nkx * MT; i += SK_EPI_WARPS * 32)
                if (i % MT >= m) smS[i] = 0.0f;
            uint32_t bad = 0;
            // groups in batches of 4 per warp, the batch's loads issued before any is used (the
            // activations may come from DRAM: one round trip per batch, not per group)
            for (int i0 = ew; i0 < m * nkx; i0 += 4 * SK_EPI_WARPS) {
                uint32_t w[4][2];
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const int i = i0 + b * SK_EPI_WARPS;
                    w[b][0] = w[b][1] = 0u;
                    if (i < m * nkx) {
                        const int j = i / nkx, s = i - j * nkx;
                        const uint16_t* xg = p.x + int64_t(j) * p.ld_x + int64_t(kx0 + s) * 128 + 4 * lane;
                        asm volatile("ld.global.nc.v2.u32 {%0,%1}, [%2];" : "=r"(w[b][0]), "=r"(w[b][1]) : "l"(xg));
                    }
                }
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const int i = i0 + b * SK_EPI_WARPS;
                    if (i >= m * nkx) break;  // warp-uniform
                    const int j = i / nkx, s = i - j * nkx;
                    const uint32_t a2 = bmax_abs2(w[b][0], w[b][1]) & 0x7FFF7FFFu;
                    const uint32_t ab = __reduce_max_sync(0xFFFFFFFFu, max(a2 & 0xFFFFu, a2 >> 16));
                    const bool fast = ab >= kAmaxFastGuardBits && ab < kNonFiniteBits;  // warp-uniform
                    float sc, rc = 0.0f;
                    uint32_t code;
                    if (fast) {
                        table_scale_rcp(tabs, ab, sc, rc);
                        encode_words<true, 2>(w[b], sc, rc, &code);
                    } else {
                        sc = scale_from_amax_bits(ab);
                        encode_words<false, 2>(w[b], sc, 0.0f, &code);
                    }
                    const uint32_t chunk = static_cast<uint32_t>(lane >> 2) ^ static_cast<uint32_t>(j & 7);
                    asm volatile("st.shared.u32 [%0], %1;" ::"r"(smem_u32(smX + s * SkFxCfg::X_SLOT + j * 128) +
                                                               chunk * 16u + static_cast<uint32_t>(lane & 3) * 4u),
                                 "r"(code)
                                 : "memory");
                    if (lane == 0) smS[s * MT + j] = sc;
                    bad |= ab >= kNonFiniteBits ? 1u : 0u;
                }
            }
            if (bad && lane == 0 && p.flag != nullptr) *p.flag = 1;
            fence_proxy_async_smem();  // the generic-proxy code stores, before the MMA reads them
            asm volatile("bar.sync 1, %0;" ::"n"(SK_EPI_WARPS * 32) : "memory");
            if (threadIdx.x == SK_EPI_WARP0 * 32) mbar_arrive(xready);
        }
        if (threadIdx.x == SK_EPI_WARP0 * 32) FP8Q_TREC(trace_tag, 5);
        const int qd = warp & 3;                       // TMEM lane quarter of this warp
        const int h = (warp - SK_EPI_WARP0) >> 2;      // token-column half
        const int r_in = qd * 32 + lane;               // weight row within the tile
        const int j0 = h * COLS;                       // first token column of this thread
        const int jn = p.m - j0 < COLS ? p.m - j0 : COLS;  // live columns of this thread
        const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(tmem_slot);
        int parked[2] = {-1, -1};  // tiles whose partial this CTA parked (slot 0 / slot 1)
        uint32_t it = 0;
        SegIter seg;
        seg.init(p);
        int tile, kb0, kb1;
        for (int si = 0; seg.next(p, tile, kb0, kb1); ++si) {
            const float* sbp = p.sb + int64_t(tile) * p.ld_sb;
            float acc[COLS];
#pragma unroll
            for (int j = 0; j < COLS; ++j) acc[j] = 0.0f;
            float sb_next = __ldg(sbp + kb0);
            for (int kb = kb0; kb < kb1; ++kb, ++it) {
                const float sbk = sb_next;
                if (kb + 1 < kb1) sb_next = __ldg(sbp + kb + 1);
                const uint32_t stage = it % STAGES;
                const uint32_t ph = (it / STAGES) & 1u;
                const uint32_t buf = it % NBUF;
                const uint32_t bph = (it / NBUF) & 1u;
                mbar_wait(&tfull[buf], bph);
                if (!kFX) mbar_wait(&full[stage], ph);  // (already complete) orders the TMA-written scales
                tc_fence_after();
                const float* sa_s = kFX ? smS + (kb - kx0) * MT + j0 : smS + stage * SA_STRIDE + j0;
                // chunks of <= 16 columns keep the live registers at acc + one chunk
                constexpr int CH = COLS < 16 ? COLS : 16;
#pragma unroll
                for (int c = 0; c < COLS / CH; ++c) {
                    float v[CH];
                    tmem_ld_cols<CH>(tmem + (static_cast<uint32_t>(qd * 32) << 16) + buf * MT + j0 + c * CH, v);
                    tmem_wait_ld();
                    if (c + 1 == COLS / CH) {  // the partial is in registers: hand the buffer back
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&tempty[buf]);
                    }
                    const float4* sa4 = reinterpret_cast<const float4*>(sa_s + c * CH);
#pragma unroll
                    for (int j = 0; j < CH / 4; ++j) {
                        const float4 s4 = sa4[j];
                        float* a = acc + c * CH + 4 * j;
                        a[0] = __fmaf_rn(v[4 * j + 0], __fmul_rn(s4.x, sbk), a[0]);
                        a[1] = __fmaf_rn(v[4 * j + 1], __fmul_rn(s4.y, sbk), a[1]);
                        a[2] = __fmaf_rn(v[4 * j + 2], __fmul_rn(s4.z, sbk), a[2]);
                        a[3] = __fmaf_rn(v[4 * j + 3], __fmul_rn(s4.w, sbk), a[3]);
                    }
                }
                __syncwarp();
                if (!kFX && lane == 0) mbar_arrive(&sempty[stage]);  // the scales were read
            }
            const int64_t n_row = int64_t(tile) * SK_BN + r_in;
            if (p.streamk == 2) {
                // cluster split-K: the partial goes to this CTA's (now idle) weight ring as
                // red[j][row], reduced across the cluster after the cluster barrier below
                float* red = reinterpret_cast<float*>(smW) + j0 * SK_BN + r_in;
#pragma unroll
                for (int j = 0; j < COLS; ++j) red[j * SK_BN] = acc[j];
            } else if (MT <= 128 && p.streamk == 3 && kb1 < p.num_kb) {  // (M > 128: cluster mode only)
                // ordered stream-K, head of a shared tile (this CTA's first segment): park it in
                // slot 0 and flag it; the next CTA, which holds the tile's tail as its LAST
                // segment, will find it long published
                float* mine = p.ws + (int64_t(2 * blockIdx.x) * MT + j0) * SK_BN + r_in;
#pragma unroll
                for (int j = 0; j < COLS; ++j)
                    if (j < jn) mine[j * SK_BN] = acc[j];
                __threadfence();
                asm volatile("bar.sync 1, %0;" ::"n"(SK_EPI_WARPS * 32) : "memory");
                if (threadIdx.x == SK_EPI_WARP0 * 32)
                    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p.counters + tile), "r"(1) : "memory");
            } else if (MT <= 128 && p.streamk == 3 && kb0 > 0) {
                // ordered stream-K, tail of a shared tile (this CTA's last segment): head + tail
                // in CTA order, (0 + P_head) + P_tail as the atomic fixup sums it
                if (threadIdx.x == SK_EPI_WARP0 * 32) {
                    int f = 0;
                    for (;;) {
                        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(f) : "l"(p.counters + tile) : "memory");
                        if (f != 0) break;
                        __nanosleep(64);
                    }
                    p.counters[tile] = 0;  // reusable workspace
                }
                asm volatile("bar.sync 1, %0;" ::"n"(SK_EPI_WARPS * 32) : "memory");
                const int c_head = sk_cta_of(p, int64_t(tile) * p.num_kb);
                const float* src = p.ws + (int64_t(2 * c_head) * MT + j0) * SK_BN + r_in;
                float v[COLS];
#pragma unroll
                for (int j = 0; j < COLS; ++j) v[j] = __ldcg(src + j * SK_BN);
#pragma unroll
                for (int j = 0; j < COLS; ++j) acc[j] = (0.0f + v[j]) + acc[j];
                if (n_row < p.n) sk_store(p, n_row, j0, jn, acc);
            } else if (kb0 > 0 || kb1 < p.num_kb) {
                // partial tile (first or last segment of this CTA's range): park it, no wait
                const int slot = si == 0 ? 0 : 1;
                parked[slot] = tile;
                float* mine = p.ws + (int64_t(2 * blockIdx.x + slot) * MT + j0) * SK_BN + r_in;
#pragma unroll
                for (int j = 0; j < COLS; ++j) {
                    if (j < jn) *mine = acc[j];
                    mine += SK_BN;
                }
            } else if (n_row < p.n) {
                sk_store(p, n_row, j0, jn, acc);
            }
        }
        if (threadIdx.x == SK_EPI_WARP0 * 32) FP8Q_TREC(trace_tag, 6);
        // ---- stream-K fixup of the parked tiles (at most two per CTA): one fence, both
        // counters bumped in one round trip, then the sums of the tiles this CTA completes
        if (parked[0] >= 0 || parked[1] >= 0) {
            __shared__ int sk_last[2];
            __threadfence();
            asm volatile("bar.sync 1, %0;" ::"n"(SK_EPI_WARPS * 32) : "memory");
            if (threadIdx.x == SK_EPI_WARP0 * 32) {
                int old[2] = {-1, -1};
#pragma unroll
                for (int slot = 0; slot < 2; ++slot)
                    if (parked[slot] >= 0) old[slot] = atomicAdd(&p.counters[parked[slot]], 1);
                __threadfence();
#pragma unroll
                for (int slot = 0; slot < 2; ++slot) {
                    const int t = parked[slot];
                    const int64_t t0 = int64_t(t) * p.num_kb;
                    sk_last[slot] = t >= 0 && old[slot] == sk_cta_of(p, t0 + p.num_kb - 1) - sk_cta_of(p, t0);
                }
            }
            asm volatile("bar.sync 1, %0;" ::"n"(SK_EPI_WARPS * 32) : "memory");
#pragma unroll 1
            for (int slot = 0; slot < 2; ++slot) {
                if (!sk_last[slot]) continue;
                const int t = parked[slot];
                const int64_t t0 = int64_t(t) * p.num_kb;
                const int c_first = sk_cta_of(p, t0);
                const int c_last = sk_cta_of(p, t0 + p.num_kb - 1);
                // CTA c parked tile t in slot 0 if t is the first tile of c's range, else slot 1.
                // Unpredicated loads (columns past m hold stale values that are never stored)
                // so each CTA's whole row segment is in flight at once.
                // The contributors' partials are fetched FC CTAs at a time (all loads of a group in
                // flight together: one L2 round trip per group, not one per contributing CTA --
                // the per-CTA timeline showed the fixup CTAs exiting ~8 us after their stream
                // ended with one dependent round trip per contributor) and summed in CTA order,
                // so the result is bit-identical to the one-at-a-time sum.
                constexpr int FC_REGS = 64;
                constexpr int FC = COLS >= FC_REGS ? 1 : FC_REGS / COLS;
                float acc[COLS];
#pragma unroll
                for (int j = 0; j < COLS; ++j) acc[j] = 0.0f;
#pragma unroll 1
                for (int cg = c_first; cg <= c_last; cg += FC) {
                    float v[FC][COLS];
#pragma unroll
                    for (int f = 0; f < FC; ++f) {
                        const int c = cg + f;
                        if (FC == 1 || c <= c_last) {
                            const int64_t c_start = int64_t(c) * p.total / gridDim.x;
                            const float* src =
                                p.ws + (int64_t(2 * c + (c_start < t0 ? 1 : 0)) * MT + j0) * SK_BN + r_in;
#pragma unroll
                            for (int j = 0; j < COLS; ++j) v[f][j] = __ldcg(src + j * SK_BN);
                        }
                    }
#pragma unroll
                    for (int f = 0; f < FC; ++f)
                        if (FC == 1 || cg + f <= c_last) {
#pragma unroll
                            for (int j = 0; j < COLS; ++j) acc[j] += v[f][j];
                        }
                }
                if (threadIdx.x == SK_EPI_WARP0 * 32) p.counters[t] = 0;  // reusable workspace
                const int64_t n_row = int64_t(t) * SK_BN + r_in;
                if (n_row < p.n) sk_store(p, n_row, j0, jn, acc);
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (p.streamk == 2) {
        // ---- cluster split-K reduction: every CTA of the cluster parked its [MT][128] fp32
        // partial in its own shared memory; CTA r sums elements [r E/cs, (r+1) E/cs) of the
        // E = m x 128 live ones over the cluster's CTAs IN RANK ORDER (deterministic), reading
        // the peers' shared memory through DSMEM, and stores them.  No global workspace, no
        // fences, no atomics.
        cluster_sync_all();
        {  // all 12 warps (the control warps' 72 registers hold one unit's cs loads)
            grid_dependency_wait();
            const uint32_t rank = cluster_ctarank();
            const int tile = static_cast<int>(blockIdx.x) / p.cs;
            // units of 4 consecutive weight rows of one token column: one 16-byte DSMEM load per
            // peer (scalar remote loads were measured at ~4 B/cycle: 6 us for a 128 x 128 tile)
            const int U = p.m * (SK_BN / 4);
            const int u1 = static_cast<int>((int64_t(rank) + 1) * U / p.cs);
            const uint32_t red0 = smem_u32(smW);
            const int te = threadIdx.x;
            constexpr int RU = 1;  // units per thread per pass (all cs loads of a unit in flight together)
            for (int q0 = static_cast<int>(int64_t(rank) * U / p.cs) + te; q0 < u1; q0 += RU * SK_THREADS) {
                float4 v[RU][8];
#pragma unroll
                for (int r = 0; r < RU; ++r) {
                    const int q = q0 + r * SK_THREADS;
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        if (c < p.cs && q < u1) {
                            uint32_t ra;
                            asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(red0 + 16u * q), "r"(c));
                            asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];"
                                         : "=f"(v[r][c].x), "=f"(v[r][c].y), "=f"(v[r][c].z), "=f"(v[r][c].w)
                                         : "r"(ra));
                        }
                    }
                }
#pragma unroll
                for (int r = 0; r < RU; ++r) {
                    const int q = q0 + r * SK_THREADS;
                    if (q >= u1) break;
                    float4 sum = v[r][0];
#pragma unroll
                    for (int c = 1; c < 8; ++c)
                        if (c < p.cs) {
                            sum.x += v[r][c].x;
                            sum.y += v[r][c].y;
                            sum.z += v[r][c].z;
                            sum.w += v[r][c].w;
                        }
                    const int j = q / (SK_BN / 4), row = 4 * (q - j * (SK_BN / 4));
                    const int64_t n_row = int64_t(tile) * SK_BN + row;
                    const float sv[4] = {sum.x, sum.y, sum.z, sum.w};
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        if (n_row + t < p.n) {
                            if (p.out_f32)
                                static_cast<float*>(p.d)[int64_t(j) * p.ld_d + n_row + t] = sv[t];
                            else
                                static_cast<__nv_bfloat16*>(p.d)[int64_t(j) * p.ld_d + n_row + t] =
                                    __float2bfloat16_rn(sv[t]);
                        }
                    }
                }
            }
        }
        cluster_sync_all();  // no CTA leaves while a peer may still read its shared memory
    }
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(*reinterpret_cast<volatile uint32_t*>(tmem_slot), C::TMEM_COLS);
    }
    if (threadIdx.x == SK_EPI_WARP0 * 32) FP8Q_TREC(trace_tag, 7);
}

// ------------------------------------------------------------------------------ host side
int sk_mt(int64_t m) { return m <= 16 ? 16 : m <= 32 ? 32 : m <= 64 ? 64 : m <= 128 ? 128 : 256; }

// Stream-K grid: one CTA per SM, but at least 2 k-blocks per CTA.
int64_t sk_grid(int64_t tiles, int64_t num_kb, int sms) {
    const int64_t total = tiles * num_kb;
    int64_t g = std::min<int64_t>(sms, total / 2);
    return g < 1 ? 1 : g;
}
bool sk_streamk_possible(int64_t n, int64_t k, int sms) {
    const int64_t tiles = (n + SK_BN - 1) / SK_BN;
    return tiles * 4 <= static_cast<int64_t>(SK_COUNTER_BYTES) && sk_grid(tiles, k / SK_BK, sms) > 1;
}
size_t sk_ws_bytes(int64_t m, int64_t n, int64_t k, int sms) {
    if (m > 128 || !sk_streamk_possible(n, k, sms)) return 0;  // M > 128: cluster split-K only
    const int64_t tiles = (n + SK_BN - 1) / SK_BN;
    return SK_COUNTER_BYTES + static_cast<size_t>(2 * sk_grid(tiles, k / SK_BK, sms)) * sk_mt(m) * SK_BN * 4;
}

struct SkDev {
    int sms = 0;
    bool attr_set = false;
};
SkDev g_sk_dev[64];
std::mutex g_sk_mu;

cudaError_t sk_device_info(int& sms) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lk(g_sk_mu);
    SkDev& di = g_sk_dev[dev];
    if (!di.attr_set) {
        e = cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, dev);
        if (e != cudaSuccess) return e;
#define SK_ATTR(MT)                                                                                  \
    e = cudaFuncSetAttribute(fp8_gemm_skinny_kernel<MT>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             static_cast<int>(SkCfg<MT>::SMEM_BYTES));                                \
    if (e != cudaSuccess) return e;
        SK_ATTR(16)
        SK_ATTR(32)
        SK_ATTR(64)
        SK_ATTR(128)
        SK_ATTR(256)
#undef SK_ATTR
        e = cudaFuncSetAttribute(fp8_gemm_skinny_kernel<16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(SkFxCfg::SMEM_BYTES));
        if (e != cudaSuccess) return e;
        di.attr_set = true;
    }
    sms = di.sms;
    return cudaSuccess;
}

// Cluster split-K (mode 2) applies when whole weight tiles would leave at least half the SMs
// idle: the largest cs <= 8 with tiles * cs <= sms whose clusters are all co-resident
// (cudaOccupancyMaxActiveClusters: a cluster must fit in one GPC).  0: not applicable.
// Dev override FP8Q_SKINNY_CLUSTER=0 disables it (stream-K instead).  Cached per shape class.
template <int MT>
int sk_cluster_size(int tiles, int num_kb, int sms) {
    static const bool enabled = [] {
        const char* e = std::getenv("FP8Q_SKINNY_CLUSTER");
        return !(e != nullptr && e[0] == '0');
    }();
    if (!enabled || tiles * 2 > sms || num_kb < 4) return 0;
    struct Entry { int tiles, num_kb, sms, cs; };
    static Entry cache[32];
    static int used = 0;
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    for (int i = 0; i < used; ++i)
        if (cache[i].tiles == tiles && cache[i].num_kb == num_kb && cache[i].sms == sms) return cache[i].cs;
    int c = std::min(8, std::min(sms / tiles, num_kb / 2));
    for (; c >= 2; --c) {
        cudaLaunchConfig_t q = {};
        q.gridDim = dim3(static_cast<unsigned>(tiles * c));
        q.blockDim = dim3(SK_THREADS);
        q.dynamicSmemBytes = SkCfg<MT>::SMEM_BYTES;
        cudaLaunchAttribute ca;
        ca.id = cudaLaunchAttributeClusterDimension;
        ca.val.clusterDim.x = static_cast<unsigned>(c);
        ca.val.clusterDim.y = 1;
        ca.val.clusterDim.z = 1;
        q.attrs = &ca;
        q.numAttrs = 1;
        int active = 0;
        const cudaError_t e = cudaOccupancyMaxActiveClusters(&active, fp8_gemm_skinny_kernel<MT>, &q);
        if (e == cudaSuccess && active >= tiles) break;
        cudaGetLastError();
    }
    const int cs = c >= 2 ? c : 0;
    if (used < 32) cache[used++] = Entry{tiles, num_kb, sms, cs};
    return cs;
}

template <int MT>
cudaError_t sk_launch(const GemmArgs& a, PFN_cuTensorMapEncodeTiled_v12000 encode, int sms, cudaStream_t stream) {
    const bool fx = MT == 16 && a.x_bf16 != nullptr;  // fused activation quantization
    CUtensorMap tmW, tmX, tmS;
    {
        cuuint64_t dims[2] = {static_cast<cuuint64_t>(a.k), static_cast<cuuint64_t>(a.n)};
        cuuint64_t strides[1] = {static_cast<cuuint64_t>(a.ld_b)};
        cuuint32_t box[2] = {SK_BK, SK_BN};
        cuuint32_t estr[2] = {1, 1};
        if (encode(&tmW, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(a.b), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    if (fx) {  // no activation / scale tensors: the kernel reads the BF16 activations itself
        tmX = tmW;
        tmS = tmW;
    } else {
        cuuint64_t dims[2] = {static_cast<cuuint64_t>(a.k), static_cast<cuuint64_t>(a.m)};
        cuuint64_t strides[1] = {static_cast<cuuint64_t>(a.ld_a)};
        cuuint32_t box[2] = {SK_BK, MT};
        cuuint32_t estr[2] = {1, 1};
        if (encode(&tmX, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(a.a), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    if (!fx) {
        // activation scales, MN-major [k/128][ld_sa]: row kb holds the m tokens' scales
        cuuint64_t dims[2] = {static_cast<cuuint64_t>(a.m), static_cast<cuuint64_t>(a.k / SK_BK)};
        cuuint64_t strides[1] = {static_cast<cuuint64_t>(a.ld_sa * 4)};
        cuuint32_t box[2] = {MT, 1};
        cuuint32_t estr[2] = {1, 1};
        if (encode(&tmS, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(a.sa), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    SkParams p;
    p.sb = a.sb;
    p.ld_sb = a.ld_sb;
    p.d = a.d;
    p.ld_d = a.ld_d;
    p.out_f32 = a.out_f32 ? 1 : 0;
    p.m = static_cast<int>(a.m);
    p.n = static_cast<int>(a.n);
    p.num_kb = static_cast<int>(a.k / SK_BK);
    p.tiles = static_cast<int>((a.n + SK_BN - 1) / SK_BN);
    p.total = int64_t(p.tiles) * p.num_kb;
    p.streamk = 0;
    p.cs = 1;
    // Weight stages issued before griddepcontrol.wait.  Measured (decode layer, A/B x2, session 3):
    // the whole ring (11 stages at M = 1, 19 MB over 96 SMs for qkv) saturates HBM while the
    // preceding activation quantizer waits for its own (tiny) input behind it, so that
    // quantizer's load latency grew to ~3 us; 4 stages: M = 1 layer 66.5 -> 64.8 us, M = 64
    // 79.6 -> 78.5, M >= 128 unchanged (0 / 2 / 6 stages: 68.8 / 66.6 / 64.5 at M = 1).
    // Dev A/B: FP8Q_SKINNY_PREFETCH=n.
    static const int prefetch = [] {
        const char* e = std::getenv("FP8Q_SKINNY_PREFETCH");
        return e ? std::atoi(e) : 4;
    }();
    p.prefetch = prefetch;
    p.x = fx ? a.x_bf16 : nullptr;
    p.ld_x = a.ld_x;
    p.flag = a.nonfinite_flag;
    p.ws = nullptr;
    p.counters = nullptr;
    unsigned grid = static_cast<unsigned>(std::min<int64_t>(p.tiles, sms));  // whole tiles
    const size_t need = sk_ws_bytes(a.m, a.n, a.k, sms);
    if (need > 0 && a.workspace != nullptr && a.workspace_bytes >= need) {
        p.streamk = 1;
        p.counters = static_cast<int32_t*>(a.workspace);
        p.ws = reinterpret_cast<float*>(static_cast<char*>(a.workspace) + SK_COUNTER_BYTES);
        grid = static_cast<unsigned>(sk_grid(p.tiles, p.num_kb, sms));
        static const bool ordered = [] {  // dev A/B: FP8Q_SKINNY_ORDERED=0 keeps the atomic fixup
            const char* e = std::getenv("FP8Q_SKINNY_ORDERED");
            return !(e != nullptr && e[0] == '0');
        }();
        // every range spans >= one tile's k-blocks, so each tile has at most two CTAs: the
        // ordered form (no atomics, the shared heads published at the start)
        if (ordered && p.total / grid >= p.num_kb) p.streamk = 3;
    }
    const int cs = sk_cluster_size<MT>(p.tiles, p.num_kb, sms);
    if (cs >= 2) {
        p.streamk = 2;
        p.cs = cs;
        grid = static_cast<unsigned>(p.tiles * cs);
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(SK_THREADS);
    cfg.dynamicSmemBytes = fx ? SkFxCfg::SMEM_BYTES : SkCfg<MT>::SMEM_BYTES;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    static const int no_pdl = [] {  // dev A/B: FP8Q_SKINNY_NOPDL=1 launches without PDL
        const char* e = std::getenv("FP8Q_SKINNY_NOPDL");
        return (e != nullptr && e[0] == '1') ? 1 : 0;
    }();
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = no_pdl ? 0 : 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = static_cast<unsigned>(p.cs);
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    if constexpr (MT == 16) {
        if (fx) return cudaLaunchKernelEx(&cfg, fp8_gemm_skinny_kernel<16, true>, tmW, tmX, tmS, p);
    }
    return cudaLaunchKernelEx(&cfg, fp8_gemm_skinny_kernel<MT>, tmW, tmX, tmS, p);
}

}  // namespace

bool skinny_gemm_applies(const GemmArgs& a) {
    static const int forced = [] {
        const char* e = std::getenv("FP8Q_GEMM_KIND");
        return e ? std::atoi(e) : 0;
    }();
    if (forced != 0 && forced != 16) return false;  // dev override: 16 = skinny, others = gemm.cu kinds
    if (a.offsets != nullptr || a.m < 1 || a.m > kSkinnyMaxM || (reinterpret_cast<uintptr_t>(a.sa) & 15u) != 0 ||
        (a.ld_sa % 4) != 0)
        return false;
    // Measured (tools/kernel_bench.py --decode --graph, Qwen3-8B shapes): up to M = 32 this
    // kernel wins everywhere; above, the 128 x 256 tile kernel wins once it has >= 64 tiles to
    // spread (gate_up), this one where the tile kernel would leave most SMs idle (qkv, o, down).
    if (a.m > 128) {  // M = 129..256: only as cluster split-K (few weight tiles, e.g. o/down/qkv)
        if (forced == 16) return true;
        // ... unless the CTA pair splits its tiles along K over most SMs (M = 256: qkv, down)
        if (a.workspace != nullptr && pair_tail_split_applies(a.m, a.n, a.k, a.workspace_bytes)) return false;
        int sms = 0;
        if (sk_device_info(sms) != cudaSuccess) return false;
        return sk_cluster_size<256>(static_cast<int>((a.n + SK_BN - 1) / SK_BN), static_cast<int>(a.k / SK_BK), sms) >= 2;
    }
    return forced == 16 || a.m <= 32 || (a.n + 255) / 256 < 64;
}

bool skinny_fused_act_applies(const GemmArgs& a) {
    static const bool enabled = [] {  // dev A/B: FP8Q_LINEAR_FUSED=0 keeps quantizer + GEMM launches
        const char* e = std::getenv("FP8Q_LINEAR_FUSED");
        return !(e != nullptr && e[0] == '0');
    }();
    if (!enabled || a.m < 1 || a.m > 16 || a.k % SK_BK != 0 || !skinny_gemm_applies(a)) return false;
    int sms = 0;
    if (sk_device_info(sms) != cudaSuccess) return false;
    const int tiles = static_cast<int>((a.n + SK_BN - 1) / SK_BN);
    const int num_kb = static_cast<int>(a.k / SK_BK);
    const int cs = sk_cluster_size<16>(tiles, num_kb, sms);
    // the CTA's activation k-blocks must fit the kFxSlots code slots (sk_fx_range)
    if (cs >= 2) return (num_kb + cs - 1) / cs <= kFxSlots;
    return num_kb <= kFxSlots;
}

size_t skinny_workspace_bytes(int64_t m, int64_t n, int64_t k) {
    int sms = 0;
    if (sk_device_info(sms) != cudaSuccess) sms = 148;
    return sk_ws_bytes(m, n, k, sms);
}

cudaError_t launch_fp8_gemm_skinny(const GemmArgs& a, void* encode_fn, cudaStream_t stream) {
    auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(encode_fn);
    if (encode == nullptr) return cudaErrorNotSupported;
    int sms = 0;
    cudaError_t e = sk_device_info(sms);
    if (e != cudaSuccess) return e;
    switch (sk_mt(a.m)) {
        case 16: return sk_launch<16>(a, encode, sms, stream);
        case 32: return sk_launch<32>(a, encode, sms, stream);
        case 64: return sk_launch<64>(a, encode, sms, stream);
        case 128: return sk_launch<128>(a, encode, sms, stream);
        default: return sk_launch<256>(a, encode, sms, stream);
    }
}

}  // namespace fp8q

FP8Q_TRACE_DUMP_FN(fp8q_trace_dump_skinny)
