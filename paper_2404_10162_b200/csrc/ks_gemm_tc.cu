// ks_gemm_tc.cu -- the LSTM gate GEMM on the 5th-generation tensor cores
// (tcgen05 + TMEM + TMA), with the LSTM cell fused into the epilogue.
//
//   gates[M x 4H] = A[M x K] . W^T + G[slot(row)]         (nn.cpp:88-128)
//   c' = sig(f) c_prev[parent(row)] + sig(i) tanh(g);  h' = sig(o) tanh(c')
//
// Precision modes (include/ks_b200.h):
//   F16X3: 2^8 A = A_hi + A_lo and 2^8 W = W_hi + W_lo (fp16 planes, ~22-bit
//          operands).  One TMEM accumulator collects A_hi.W_hi + A_hi.W_lo +
//          A_lo.W_hi (three MMAs per K step); gates = 2^-16 D.  The dropped
//          A_lo.W_lo term is ~2^-22 relative.
//   BF16:  one bf16 MMA per K step (A_hi / W_hi planes hold bf16).
//
// Structure: persistent CTAs (one per SM), 384 threads:
//   warp 0      TMA producer (A and W tiles, 128B swizzle, mbarrier ring)
//   warp 1      MMA issuer (one elected thread, tcgen05.mma.cta_group::1)
//   warp 2      TMEM allocator
//   warps 4..11 epilogue: tcgen05.ld -> cell update -> h, c (+ split h) stores
// Tile: 128 rows x (4 gates x UNITS hidden units); the weight packing
// interleaves the gates per UNITS-unit block so one N tile holds i,f,o,g of the
// same units and the cell update needs no cross-CTA exchange.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstdio>

#include "ks_common.cuh"
#include "ks_tc.cuh"

namespace ksb {


struct TcProblem {
    LstmArgs p;
    int m_tiles;
    int n_tiles;
    int k_blocks;
    int tile_begin;  // first global tile index of this problem
    int tma_out;     // h / c of whole 32-row warp slices leave through bulk tensor stores
    alignas(64) CUtensorMap mh;  // fp32 [M][H] views of h_out / c_out, box 32 rows x 8 units
    alignas(64) CUtensorMap mc;
    int tma_a;                   // the split copy of h (hA_hi / hA_lo) through bulk stores too
    alignas(64) CUtensorMap mah; // fp16 [M][H] views of hA_hi / hA_lo, box 32 rows x 8 units
    alignas(64) CUtensorMap mal;
};

// alpha-block mode: K-blocks of one tile.  The B operand's P^T columns start at
// x0 = 7 * b0 rounded down to 8 (TMA tile loads need 16-byte aligned inner
// coordinates) and end after the tile's last config; the A operand keeps
// kb_alpha (max) alpha blocks, of which the tile contracts the first kba_t.
struct TileK {
    int kba_t;  // alpha K-blocks this tile contracts
    int x0;     // first P^T column
    int nkb;    // total K-blocks of the tile
};
// mt indexes alpha tiles of TR rows (<= 128 -- config-aligned tiles hold whole
// configs -- or 256 = one CTA pair); compacted rows (cp_cfg): the tile's first and
// last configs come from the row -> config map, Mv = the rows of the launch
__device__ __forceinline__ TileK tile_k(const LstmArgs& p, int k_blocks, int mt, int TR, int Mv) {
    TileK r{0, 0, k_blocks};
    if (p.kb_alpha > 0) {
        int b0, b1;
        if (p.cp_cfg) {
            const int last = (mt * TR + TR < Mv ? mt * TR + TR : Mv) - 1;
            b0 = p.cp_cfg[mt * TR];
            b1 = p.cp_cfg[last];
        } else {
            b0 = (mt * TR) / p.rows_per_cfg;
            b1 = (mt * TR + TR - 1) / p.rows_per_cfg;
        }
        r.x0 = (7 * b0) & ~7;
        r.kba_t = (7 * (b1 + 1) - r.x0 + kTcBK - 1) / kTcBK;
        if (r.kba_t > p.kb_alpha) r.kba_t = p.kb_alpha;
        r.nkb = k_blocks - p.kb_alpha + r.kba_t;
    }
    return r;
}

struct TcParams {
    TcProblem prob[2];
    int n_prob;
    int total_tiles;
};

constexpr int TC_BM = 128;
constexpr int TC_BK = kTcBK;

// CG = 2: a CTA pair (cluster of 2 on one TPC) runs M = 256 MMAs with
// tcgen05.mma.cta_group::2: each CTA holds its 128 A rows and HALF of the B tile
// (BN/2 gate rows), so per-SM shared-memory operand traffic drops by a third;
// only the leader CTA issues MMAs.
template <int UNITS, bool SPLIT, int CG = 1>
struct TcCfg {
    static constexpr int BN = 4 * UNITS;                       // gate columns per tile
    static constexpr int PLANES = SPLIT ? 2 : 1;
    static constexpr int A_BYTES = TC_BM * TC_BK * 2;          // one plane
    static constexpr int B_BYTES = (BN / CG) * TC_BK * 2;      // this CTA's share of one plane
    static constexpr int STAGE_BYTES = PLANES * (A_BYTES + B_BYTES);
    static constexpr int ACC_COLS = BN;                        // fp32 TMEM columns per accumulator
    static constexpr int ACC_STAGES = 512 / ACC_COLS >= 2 ? 2 : 1;
    static constexpr int STAGES = (200 * 1024) / STAGE_BYTES > 6 ? 6 : (200 * 1024) / STAGE_BYTES;
    // output staging for the bulk h / c stores: 8 epilogue warps x 2 buffers x (h, c) x 32 rows x 8 units
    static constexpr int OUT_STAGE = 8 * 2 * 2 * 32 * 8 * 4;
    static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /* align */ + 256 /* barriers */ + OUT_STAGE;
    // instruction descriptor: fp32 accumulate (bits 4-5 = 1), A/B fp16 (0) or bf16 (1) at
    // bits 7-9 / 10-12, both K-major, N >> 3 at bits 17-22, M >> 4 at bits 24-28
    static constexpr uint32_t IDESC = (1u << 4) | ((SPLIT ? 0u : 1u) << 7) | ((SPLIT ? 0u : 1u) << 10) |
                                      ((uint32_t)(BN >> 3) << 17) | ((uint32_t)((CG * TC_BM) >> 4) << 24);
};

// Cell nonlinearities with MUFU exp2 + fast reciprocal: absolute error ~1e-7,
// far below the fp32-grade GEMM tolerance (the FP32 mode keeps libm expf/tanhf).
// The LSTM cell (nn.cpp:88-128) with 5 exp2 + 2 reciprocals on the MUFU pipe instead
// of 5 + 5: with A = 1 + e^-f, B = 1 + e^-i, G = 1 + e^2g (sig(f) = 1/A, sig(i) = 1/B,
// tanh(g) = (G - 2)/G),  c' = (c B G + A (G - 2)) / (A B G);  with O = 1 + e^-o and
// Q = 1 + e^2c',  h' = (Q - 2) / (O Q).  Arguments are clamped so the products stay
// finite (|sig, tanh| saturate to within 1.4e-11 of their limits there, far below
// the fp32 resolution of the states).
__device__ __forceinline__ void lstm_cell_fast(float zi, float zf, float zo, float zg, float cp, float& c,
                                               float& h) {
    const float A = 1.0f + __expf(-fminf(fmaxf(zf, -25.0f), 25.0f));
    const float B = 1.0f + __expf(-fminf(fmaxf(zi, -25.0f), 25.0f));
    const float G = 1.0f + __expf(2.0f * fminf(fmaxf(zg, -12.5f), 12.5f));
    c = __fdividef(fmaf(cp * B, G, A * (G - 2.0f)), A * B * G);
    const float O = 1.0f + __expf(-fminf(fmaxf(zo, -25.0f), 25.0f));
    const float Q = 1.0f + __expf(2.0f * fminf(fmaxf(c, -12.5f), 12.5f));
    h = __fdividef(Q - 2.0f, O * Q);
}

// Cell-mode epilogue of one accumulator (rows row0 + [q*32, q*32+32) of the tile,
// units [half*UNITS/2, +UNITS/2) of N tile nt).  bars[tfull + acc] / bars[tempty + acc]:
// the accumulator's full / empty barriers.  Each 16-row group g of the warp's 32
// rows is read with tcgen05.ld.16x256b: lane t holds rows t/4 and t/4 + 8 of the
// group, units 2(t%4), 2(t%4)+1 of each 8-unit chunk, all four gates (one load per
// gate block) -- the LSTM cell needs no exchange, and the 4 lanes of a quad write
// one row's 8 units (a whole 32-byte segment) per store instruction.
template <int UNITS, bool SPLIT, int CG>
__device__ __forceinline__ void epilogue_cells(const LstmArgs& p, uint64_t* bars, uint32_t tmem_base, int acc,
                                               uint32_t acc_phase, int row0, int TRp, int nt, int q, int half,
                                               int lane, int tfull, int tempty, int acc_cols, bool leader,
                                               const TcProblem& pr, float* stg, int& stg_buf) {
    constexpr int HU = UNITS / 2;
    constexpr int NCH = HU / 8;
    const int tq = lane >> 2, tcol = 2 * (lane & 3);
    int rows[4], slots[4], crows[4];
    bool valid[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {  // i = 2 g + j: group g, row t/4 + 8 j
        const int lr = q * 32 + 16 * (i >> 1) + tq + 8 * (i & 1);
        rows[i] = row0 + lr;
        valid[i] = rows[i] < p.M && (CG == 2 || lr < TRp);
        slots[i] = valid[i] ? p.slot_base + (p.slot_ptr ? p.slot_ptr[(long long)rows[i] * p.slot_stride] : 0) : 0;
        crows[i] = valid[i] ? (p.parent ? p.parent[rows[i]] : rows[i]) : -1;
    }
    const bool have_cprev = p.c_prev != nullptr;
    // bulk stores only for warp slices whose 32 rows all belong to this tile
    const bool bulk = pr.tma_out && row0 + q * 32 + 31 < p.M && (CG == 2 || q * 32 + 31 < TRp);
    // G[slot] and c_prev of the chunk's 2 units per row, prefetched a chunk ahead
    float2 gn[4][4], cn[4];
    auto load_bc = [&](int c, float2 (&gx)[4][4], float2 (&cx)[4]) {
        const int u0 = nt * UNITS + half * HU + c * 8 + tcol;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float* G = p.G + (long long)slots[i] * 4 * p.H;
#pragma unroll
            for (int gt = 0; gt < 4; ++gt)
                gx[i][gt] = valid[i] ? *reinterpret_cast<const float2*>(G + gt * p.H + u0) : make_float2(0.f, 0.f);
            cx[i] = (valid[i] && have_cprev && crows[i] >= 0)
                        ? *reinterpret_cast<const float2*>(p.c_prev + (long long)crows[i] * p.ldc_prev + u0)
                        : make_float2(0.f, 0.f);
        }
    };
    load_bc(0, gn, cn);
    tc::mbar_wait(tc::smem_u32(&bars[tfull + acc]), acc_phase);
    tc::fence_after();
    const uint32_t tq_base = tmem_base + ((uint32_t)(q * 32) << 16) + acc * acc_cols;
    constexpr float sc = SPLIT ? kSplitUnscale : 1.0f;  // a power of two: exact
    const float2 sc2 = make_float2(sc, sc);
#pragma unroll 1
    for (int c = 0; c < NCH; ++c) {
        const int uc = half * HU + c * 8;
        float v[2][4][4];  // [group][gate][r0u0, r0u1, r1u0, r1u1]
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
            for (int gt = 0; gt < 4; ++gt)
                tc::tmem_ld16x256(tq_base + ((uint32_t)(16 * g) << 16) + gt * UNITS + uc, v[g][gt]);
        tc::tmem_wait_ld();
        if (c == NCH - 1) {  // this warp's TMEM reads are done: release the accumulator
            tc::fence_before();
            __syncwarp();
            if (lane == 0) {
                if (CG == 2 && !leader)
                    tc::mbar_arrive_remote(tc::smem_u32(&bars[tempty + acc]), 0);
                else
                    tc::mbar_arrive(tc::smem_u32(&bars[tempty + acc]));
            }
        }
        const int u0 = nt * UNITS + uc + tcol;
        // the 8 cells of the chunk (4 rows x 2 units) computed unconditionally and
        // interleaved (independent dependency chains), stores predicated per row
        float hv[4][2], cv[4][2];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int g = i >> 1, j = i & 1;
            float2 z[4];
#pragma unroll
            for (int gt = 0; gt < 4; ++gt)
                z[gt] = __ffma2_rn(make_float2(v[g][gt][2 * j], v[g][gt][2 * j + 1]), sc2, gn[i][gt]);
            lstm_cell_fast(z[0].x, z[1].x, z[2].x, z[3].x, cn[i].x, cv[i][0], hv[i][0]);
            lstm_cell_fast(z[0].y, z[1].y, z[2].y, z[3].y, cn[i].y, cv[i][1], hv[i][1]);
        }
        // the next chunk's G[slot] / c_prev, in flight during this chunk's stores and the
        // next chunk's TMEM loads (one register set: these loads reuse gn / cn)
        if (c + 1 < NCH) load_bc(c + 1, gn, cn);
        const bool bulk_a = bulk && pr.tma_a;
        if (bulk) {
            // the warp's 32 x 8 slice of h and c (and of the split h, the encoder's next
            // operand) through shared memory and bulk tensor stores (one engine
            // transaction per slice instead of 64 row-segment stores); with the split
            // planes the 3 KB slice set is single-buffered
            float* sh = bulk_a ? stg : stg + stg_buf * 512;
            float* scb = sh + 256;
            __half* sah = reinterpret_cast<__half*>(sh + 512);
            __half* sal = sah + 256;
            if (lane == 0) {
                if (bulk_a)
                    tc::bulk_wait_read<0>();
                else
                    tc::bulk_wait_read<1>();  // the group that last read this buffer is done
            }
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int lr = 16 * (i >> 1) + tq + 8 * (i & 1);
                *reinterpret_cast<float2*>(sh + lr * 8 + tcol) = make_float2(hv[i][0], hv[i][1]);
                *reinterpret_cast<float2*>(scb + lr * 8 + tcol) = make_float2(cv[i][0], cv[i][1]);
                if (bulk_a) {
                    __half2 hh, hl;
                    split_f16x2(hv[i][0], hv[i][1], hh, hl);
                    *reinterpret_cast<__half2*>(sah + lr * 8 + tcol) = hh;
                    *reinterpret_cast<__half2*>(sal + lr * 8 + tcol) = hl;
                }
            }
            tc::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
                tc::tma_store_2d(&pr.mh, tc::smem_u32(sh), nt * UNITS + uc, row0 + q * 32);
                tc::tma_store_2d(&pr.mc, tc::smem_u32(scb), nt * UNITS + uc, row0 + q * 32);
                if (bulk_a) {
                    tc::tma_store_2d(&pr.mah, tc::smem_u32(sah), nt * UNITS + uc, row0 + q * 32);
                    tc::tma_store_2d(&pr.mal, tc::smem_u32(sal), nt * UNITS + uc, row0 + q * 32);
                }
                tc::bulk_commit();
            }
            if (!bulk_a) stg_buf ^= 1;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (!valid[i]) continue;
            const long long r = rows[i];
            if (!bulk) {
                // streaming (evict-first) stores: h and c are re-read once, by the next kernels,
                // and would otherwise push the GEMM's reused operands (W, P^T) out of L2
                __stcs(reinterpret_cast<float2*>(p.h_out + r * p.ldh + u0), make_float2(hv[i][0], hv[i][1]));
                __stcs(reinterpret_cast<float2*>(p.c_out + r * p.ldc + u0), make_float2(cv[i][0], cv[i][1]));
            }
            if (p.h_out2 != nullptr)
                __stcs(reinterpret_cast<float2*>(p.h_out2 + r * p.ldh2 + u0), make_float2(hv[i][0], hv[i][1]));
            if (bulk_a) continue;  // the split h went out with the bulk stores
            if (p.hA_hi != nullptr && p.ha_bf16) {
                *reinterpret_cast<__nv_bfloat162*>(p.hA_hi + r * p.ldha + u0) =
                    __floats2bfloat162_rn(hv[i][0], hv[i][1]);
            } else if (p.hA_hi != nullptr) {
                __half2 hh, hl;
                split_f16x2(hv[i][0], hv[i][1], hh, hl);
                *reinterpret_cast<__half2*>(p.hA_hi + r * p.ldha + u0) = hh;
                *reinterpret_cast<__half2*>(p.hA_lo + r * p.ldha + u0) = hl;
            }
        }
    }
}

// Fan-out cell epilogue: the GEMM ran on PARENT rows (children of one parent share
// [ctx | h_prev] and c_prev and differ only by the fed-back token's one-hot row,
// i.e. by G[slot]); each parent row's pre-activations D serve its `fan` children:
// gates(child) = D + G[slot(child)], c_prev = the parent's c.  Layout as
// epilogue_cells (16x256b loads: a quad of lanes = one row, 8 units).
template <int UNITS, bool SPLIT, int CG>
__device__ __forceinline__ void epilogue_fan(const LstmArgs& p, uint64_t* bars, uint32_t tmem_base, int acc,
                                             uint32_t acc_phase, int row0, int TRp, int nt, int q, int half,
                                             int lane, int tfull, int tempty, int acc_cols, bool leader,
                                             const TcProblem& pr, float* stg, int& stg_buf) {
    constexpr int HU = UNITS / 2;
    constexpr int NCH = HU / 8;
    const int tq = lane >> 2, tcol = 2 * (lane & 3);
    const int fan = p.fan;
    int rows[4];
    bool valid[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int lr = q * 32 + 16 * (i >> 1) + tq + 8 * (i & 1);
        rows[i] = row0 + lr;
        valid[i] = rows[i] < p.M && (CG == 2 || lr < TRp);
    }
    const bool have_cprev = p.c_prev != nullptr;
    const bool bulk = pr.tma_out && row0 + q * 32 + 31 < p.M && (CG == 2 || q * 32 + 31 < TRp);
    float2 cn[4];
    auto load_c = [&](int c, float2 (&cx)[4]) {
        const int u0 = nt * UNITS + half * HU + c * 8 + tcol;
#pragma unroll
        for (int i = 0; i < 4; ++i)
            cx[i] = (valid[i] && have_cprev)
                        ? *reinterpret_cast<const float2*>(p.c_prev + (long long)rows[i] * p.ldc_prev + u0)
                        : make_float2(0.f, 0.f);
    };
    load_c(0, cn);
    tc::mbar_wait(tc::smem_u32(&bars[tfull + acc]), acc_phase);
    tc::fence_after();
    const uint32_t tq_base = tmem_base + ((uint32_t)(q * 32) << 16) + acc * acc_cols;
    constexpr float sc = SPLIT ? kSplitUnscale : 1.0f;  // a power of two: exact
    const float2 sc2 = make_float2(sc, sc);
#pragma unroll 1
    for (int c = 0; c < NCH; ++c) {
        const int uc = half * HU + c * 8;
        float v[2][4][4];
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
            for (int gt = 0; gt < 4; ++gt)
                tc::tmem_ld16x256(tq_base + ((uint32_t)(16 * g) << 16) + gt * UNITS + uc, v[g][gt]);
        tc::tmem_wait_ld();
        if (c == NCH - 1) {
            tc::fence_before();
            __syncwarp();
            if (lane == 0) {
                if (CG == 2 && !leader)
                    tc::mbar_arrive_remote(tc::smem_u32(&bars[tempty + acc]), 0);
                else
                    tc::mbar_arrive(tc::smem_u32(&bars[tempty + acc]));
            }
        }
        float2 cp[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) cp[i] = cn[i];
        if (c + 1 < NCH) load_c(c + 1, cn);
        const int u0 = nt * UNITS + uc + tcol;
        // child f of the thread's 4 rows at a time.  The 4 slots of child f+1 load while
        // child f computes, and child f's 16 G loads issue together: one load latency per
        // child instead of a slot -> G chain per row
        int sl[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
            sl[i] = (valid[i] && p.slot_ptr) ? __ldg(p.slot_ptr + (long long)rows[i] * fan * p.slot_stride) : 0;
#pragma unroll 1
        for (int f = 0; f < fan; ++f) {
            float2 gz[4][4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float* G = p.G + ((long long)(p.slot_base + sl[i]) * 4 * p.H + u0);
#pragma unroll
                for (int gt = 0; gt < 4; ++gt) gz[i][gt] = __ldg(reinterpret_cast<const float2*>(G + gt * p.H));
            }
            if (f + 1 < fan) {
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    sl[i] = (valid[i] && p.slot_ptr)
                                ? __ldg(p.slot_ptr + ((long long)rows[i] * fan + f + 1) * p.slot_stride)
                                : 0;
            }
            float hv[4][2], cv[4][2];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int g = i >> 1, j = i & 1;
                float2 z[4];
#pragma unroll
                for (int gt = 0; gt < 4; ++gt)
                    z[gt] = __ffma2_rn(make_float2(v[g][gt][2 * j], v[g][gt][2 * j + 1]), sc2, gz[i][gt]);
                lstm_cell_fast(z[0].x, z[1].x, z[2].x, z[3].x, cp[i].x, cv[i][0], hv[i][0]);
                lstm_cell_fast(z[0].y, z[1].y, z[2].y, z[3].y, cp[i].y, cv[i][1], hv[i][1]);
            }
            if (bulk) {
                // child f of the warp's 32 parents: rows (row0 + q*32 + j) * fan + f, one box
                // of the [parents][fan][H] view per array
                float* sh = stg + stg_buf * 512;
                float* scb = sh + 256;
                if (lane == 0) tc::bulk_wait_read<1>();
                __syncwarp();
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int lr = 16 * (i >> 1) + tq + 8 * (i & 1);
                    *reinterpret_cast<float2*>(sh + lr * 8 + tcol) = make_float2(hv[i][0], hv[i][1]);
                    *reinterpret_cast<float2*>(scb + lr * 8 + tcol) = make_float2(cv[i][0], cv[i][1]);
                }
                tc::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    tc::tma_store_3d(&pr.mh, tc::smem_u32(sh), nt * UNITS + uc, f, row0 + q * 32);
                    tc::tma_store_3d(&pr.mc, tc::smem_u32(scb), nt * UNITS + uc, f, row0 + q * 32);
                    tc::bulk_commit();
                }
                stg_buf ^= 1;
                if (p.hA_hi == nullptr) continue;
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                if (!valid[i]) continue;
                const long long r = (long long)rows[i] * fan + f;
                if (!bulk) {
                    __stcs(reinterpret_cast<float2*>(p.h_out + r * p.ldh + u0), make_float2(hv[i][0], hv[i][1]));
                    __stcs(reinterpret_cast<float2*>(p.c_out + r * p.ldc + u0), make_float2(cv[i][0], cv[i][1]));
                }
                // split h (the shared-prefix encoder's next operand)
                if (p.hA_hi != nullptr && p.ha_bf16) {
                    *reinterpret_cast<__nv_bfloat162*>(p.hA_hi + r * p.ldha + u0) =
                        __floats2bfloat162_rn(hv[i][0], hv[i][1]);
                } else if (p.hA_hi != nullptr) {
                    __half2 hh, hl;
                    split_f16x2(hv[i][0], hv[i][1], hh, hl);
                    *reinterpret_cast<__half2*>(p.hA_hi + r * p.ldha + u0) = hh;
                    *reinterpret_cast<__half2*>(p.hA_lo + r * p.ldha + u0) = hl;
                }
            }
        }
    }
}

// Compacted-row cell epilogue: row r of the tile is a distinct live parent
// (epilogue_fan's sharing, with a variable number of children per parent).  Per
// 8-unit chunk the warp stages its 32 parents' pre-activations in shared memory
// (4 KB, the bulk-store staging area, unused in this mode), then its 8 lane quads
// take the warp's children round-robin -- the children of consecutive rows are
// consecutive cp_child entries, so the load is balanced whatever the fan-outs --
// each child: gates = D(parent) + G[slot], c_prev = c(cp_prow[parent]), h / c at the
// child's own row.  The next round's entry, G and c_prev loads are in flight during
// a round's math.
template <int UNITS, bool SPLIT, int CG>
__device__ __forceinline__ void epilogue_compact(const LstmArgs& p, int Mv, uint64_t* bars, uint32_t tmem_base,
                                                 int acc, uint32_t acc_phase, int row0, int nt, int q, int grp,
                                                 int lane, int tfull, int tempty, int acc_cols, bool leader,
                                                 float* sp) {
    // 16 epilogue warps: warp (q, grp) owns TMEM lane quarter q (32 parents) and units
    // [grp * UPW, + UPW) of the tile; per 8-unit chunk and per 16-parent half (2 KB of
    // shared memory per warp) it stages the parents' scaled pre-activations, then its 8
    // lane quads take those parents' children round-robin
    constexpr int UPW = UNITS / 4;
    constexpr int NCH = UPW / 8;
    const int tq = lane >> 2, tcol = 2 * (lane & 3);
    const int wr0 = row0 + q * 32;
    int eb[3];  // children entries of the warp's parents [wr0, +16) and [wr0 + 16, +16)
#pragma unroll
    for (int g = 0; g < 3; ++g) {
        const int r = wr0 + 16 * g;
        eb[g] = r < Mv ? p.cp_cstart[r] : (Mv > wr0 ? p.cp_cstart[Mv - 1] + p.cp_ccount[Mv - 1] : 0);
    }
    if (wr0 >= Mv) eb[0] = eb[1] = eb[2] = 0;
    const bool have_cprev = p.c_prev != nullptr;
    tc::mbar_wait(tc::smem_u32(&bars[tfull + acc]), acc_phase);
    tc::fence_after();
    const uint32_t tq_base = tmem_base + ((uint32_t)(q * 32) << 16) + acc * acc_cols;
    constexpr float sc = SPLIT ? kSplitUnscale : 1.0f;
#pragma unroll 1
    for (int c = 0; c < NCH; ++c) {
        const int uc = grp * UPW + c * 8;
        float v[2][4][4];
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
            for (int gt = 0; gt < 4; ++gt)
                tc::tmem_ld16x256(tq_base + ((uint32_t)(16 * g) << 16) + gt * UNITS + uc, v[g][gt]);
        tc::tmem_wait_ld();
        if (c == NCH - 1) {
            tc::fence_before();
            __syncwarp();
            if (lane == 0) {
                if (CG == 2 && !leader)
                    tc::mbar_arrive_remote(tc::smem_u32(&bars[tempty + acc]), 0);
                else
                    tc::mbar_arrive(tc::smem_u32(&bars[tempty + acc]));
            }
        }
        const int u0 = nt * UNITS + uc + tcol;
#pragma unroll
        for (int g = 0; g < 2; ++g) {
            // parents wr0 + 16 g + [0, 16): sp[parent][gate][8 units]
            __syncwarp();  // the previous phase's readers are done
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int lr = tq + 8 * j;
#pragma unroll
                for (int gt = 0; gt < 4; ++gt)
                    *reinterpret_cast<float2*>(sp + (lr * 4 + gt) * 8 + tcol) =
                        make_float2(v[g][gt][2 * j] * sc, v[g][gt][2 * j + 1] * sc);
            }
            __syncwarp();
            const int e0 = eb[g], e1 = eb[g + 1];
            const int pr0 = wr0 + 16 * g;
            auto fetch = [&](int e, int4& en, float2 (&gz)[4], float2& cpv) {
                if (e < e1) {
                    en = __ldg(p.cp_child + e);
                    const float* G = p.G + ((long long)(p.slot_base + (en.x >= 0 ? en.y : 0)) * 4 * p.H + u0);
#pragma unroll
                    for (int gt = 0; gt < 4; ++gt) gz[gt] = __ldg(reinterpret_cast<const float2*>(G + gt * p.H));
                    cpv = (have_cprev && en.w >= 0)
                              ? *reinterpret_cast<const float2*>(p.c_prev + (long long)en.w * p.ldc_prev + u0)
                              : make_float2(0.f, 0.f);
                } else {
                    en = make_int4(-1, 0, pr0, -1);
                }
            };
            int4 en;
            float2 gz[4], cpv = make_float2(0.f, 0.f);
            fetch(e0 + tq, en, gz, cpv);
#pragma unroll 1
            for (int e = e0 + tq; e < e1; e += 8) {
                const int4 cur = en;
                float2 g4[4];
#pragma unroll
                for (int gt = 0; gt < 4; ++gt) g4[gt] = gz[gt];
                const float2 cp = cpv;
                fetch(e + 8, en, gz, cpv);
                const int lp = (unsigned)(cur.z - pr0) < 16u ? cur.z - pr0 : 0;  // dead-child entries: no store
                const float* d = sp + (lp * 4) * 8 + tcol;
                float2 z[4];
#pragma unroll
                for (int gt = 0; gt < 4; ++gt) {
                    const float2 dv = *reinterpret_cast<const float2*>(d + gt * 8);
                    z[gt] = make_float2(dv.x + g4[gt].x, dv.y + g4[gt].y);
                }
                float hv0, hv1, cv0, cv1;
                lstm_cell_fast(z[0].x, z[1].x, z[2].x, z[3].x, cp.x, cv0, hv0);
                lstm_cell_fast(z[0].y, z[1].y, z[2].y, z[3].y, cp.y, cv1, hv1);
                if (cur.x >= 0) {
                    const long long r = cur.x;
                    __stcs(reinterpret_cast<float2*>(p.h_out + r * p.ldh + u0), make_float2(hv0, hv1));
                    __stcs(reinterpret_cast<float2*>(p.c_out + r * p.ldc + u0), make_float2(cv0, cv1));
                }
            }
        }
    }
}

// CPT: the compacted-row instantiation (LstmArgs::cp_M launches only), so the
// register allocation of the other launches is not shaped by epilogue_compact
template <int UNITS, bool SPLIT, int CG, bool CPT = false>
__global__ void __launch_bounds__(CPT ? 640 : 384, 1)
    lstm_gemm_tc(const __grid_constant__ TcParams P, const __grid_constant__ CUtensorMap mA0,
                 const __grid_constant__ CUtensorMap mAl0, const __grid_constant__ CUtensorMap mB0,
                 const __grid_constant__ CUtensorMap mBl0, const __grid_constant__ CUtensorMap mA1,
                 const __grid_constant__ CUtensorMap mAl1, const __grid_constant__ CUtensorMap mB1,
                 const __grid_constant__ CUtensorMap mBl1) {
    using Cfg = TcCfg<UNITS, SPLIT, CG>;
    constexpr int S = Cfg::STAGES;
    // rows per tile of a problem: 128 (a CTA pair: 2 x 128); alpha-block launches on
    // one CTA may use config-aligned tiles of alpha_tile <= 128 rows (whole configs
    // per tile: fewer alpha columns)
    auto tile_rows = [&](const LstmArgs& a) { return (CG == 1 && a.kb_alpha > 0) ? a.alpha_tile : CG * TC_BM; };
    const int rank = CG == 2 ? (int)tc::cluster_rank() : 0;
    const bool leader = rank == 0;
    const int cid = blockIdx.x / CG, ncl = gridDim.x / CG;
    constexpr int AS = Cfg::ACC_STAGES;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * Cfg::STAGE_BYTES);
    // bars: full[S], empty[S], tfull[AS], tempty[AS]; then the TMEM base slot
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 2 * AS);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            tc::mbar_init(tc::smem_u32(&bars[s]), 1);
            tc::mbar_init(tc::smem_u32(&bars[S + s]), 1);
        }
        for (int a = 0; a < AS; ++a) {
            tc::mbar_init(tc::smem_u32(&bars[2 * S + a]), 1);
            // one arrive per epilogue warp (of the pair): 8, or 16 in the compacted instantiation
            tc::mbar_init(tc::smem_u32(&bars[2 * S + AS + a]), (CPT ? 16 : 8) * CG);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        tc::tma_prefetch(&mA0);
        tc::tma_prefetch(&mB0);
        if (SPLIT) {
            tc::tma_prefetch(&mAl0);
            tc::tma_prefetch(&mBl0);
        }
    }
    if (warp == 2) {
        if (CG == 2) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                             tc::smem_u32(tmem_slot))
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                             tc::smem_u32(tmem_slot))
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
    }
    tc::fence_before();
    __syncthreads();
    if (CG == 2) tc::cluster_sync();  // the peer's barriers are initialised before any remote arrive
    tc::fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // compacted rows (one problem): the row count is device data written by the
    // compaction before this launch; the tile loop covers ceil(Mv / TR) row tiles
    const int Mv = CPT ? *P.prob[0].p.cp_M : P.prob[0].p.M;
    int total_tiles = P.total_tiles;
    if (CPT) {
        const int tr = tile_rows(P.prob[0].p);
        const int dyn = (Mv + tr - 1) / tr * P.prob[0].n_tiles;
        total_tiles = dyn < total_tiles ? dyn : total_tiles;
    }

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = cid; t < total_tiles; t += ncl) {
                const int pi = (P.n_prob > 1 && t >= P.prob[1].tile_begin) ? 1 : 0;
                const TcProblem& pr = P.prob[pi];
                const int lt = t - pr.tile_begin;
                const int mt = lt / pr.n_tiles, nt = lt - mt * pr.n_tiles;  // mt: (pair) tile
                const int TRp = tile_rows(pr.p);
                const int arow = CG == 1 ? mt * TRp : (mt * CG + rank) * TC_BM;  // this CTA's A rows
                const int brow = nt * Cfg::BN + rank * (Cfg::BN / CG);       // this CTA's B rows
                const CUtensorMap* ma = pi ? &mA1 : &mA0;
                const CUtensorMap* mal = pi ? &mAl1 : &mAl0;
                const CUtensorMap* mb = pi ? &mB1 : &mB0;
                const CUtensorMap* mbl = pi ? &mBl1 : &mBl0;
                // alpha-block mode: B K-blocks [0, kba_t) come from P^T (held in the
                // second problem's map slots) from column x0 on (see tile_k)
                const TileK tk = tile_k(pr.p, pr.k_blocks, mt, TRp, Mv);
                for (int kb = 0; kb < tk.nkb; ++kb) {
                    tc::mbar_wait(tc::smem_u32(&bars[S + stage]), phase ^ 1);
                    const uint32_t full = tc::smem_u32(&bars[stage]);
                    // pair: the leader's barrier counts both CTAs' bytes
                    if (leader) tc::mbar_expect_tx(full, CG * Cfg::STAGE_BYTES);
                    unsigned char* st = smem + stage * Cfg::STAGE_BYTES;
                    const bool from_pt = kb < tk.kba_t;
                    // A: alpha blocks [0, kba_t), then the h columns after all kb_alpha blocks
                    const int kx = (from_pt ? kb : kb - tk.kba_t + pr.p.kb_alpha) * TC_BK;
                    const CUtensorMap* bmap = from_pt ? &mB1 : mb;
                    const CUtensorMap* blmap = from_pt ? &mBl1 : mbl;
                    const int bx = from_pt ? tk.x0 + kb * TC_BK : (kb - tk.kba_t) * TC_BK;
                    auto load = [&](uint32_t dst, const CUtensorMap* m, int x, int y) {
                        if (CG == 2)
                            tc::tma_load_2d_pair(dst, m, full, x, y);
                        else
                            tc::tma_load_2d(dst, m, full, x, y);
                    };
                    load(tc::smem_u32(st), ma, kx, arow);
                    load(tc::smem_u32(st + Cfg::A_BYTES), bmap, bx, brow);
                    if (SPLIT) {
                        load(tc::smem_u32(st + Cfg::A_BYTES + Cfg::B_BYTES), mal, kx, arow);
                        load(tc::smem_u32(st + 2 * Cfg::A_BYTES + Cfg::B_BYTES), blmap, bx, brow);
                    }
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0 && leader) {
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int t = cid; t < total_tiles; t += ncl) {
                const int pi = (P.n_prob > 1 && t >= P.prob[1].tile_begin) ? 1 : 0;
                const TcProblem& pr = P.prob[pi];
                const int mt_i = (t - pr.tile_begin) / pr.n_tiles;
                const int nkb = tile_k(pr.p, pr.k_blocks, mt_i, tile_rows(pr.p), Mv).nkb;
                tc::mbar_wait(tc::smem_u32(&bars[2 * S + AS + acc]), acc_phase ^ 1);
                tc::fence_after();
                const uint32_t d1 = tmem_base + acc * Cfg::ACC_COLS;
                for (int kb = 0; kb < nkb; ++kb) {
                    tc::mbar_wait(tc::smem_u32(&bars[stage]), phase);
                    tc::fence_after();
                    const uint32_t a0 = tc::smem_u32(smem + stage * Cfg::STAGE_BYTES);
                    const uint32_t b0 = a0 + Cfg::A_BYTES;
                    const uint32_t al = b0 + Cfg::B_BYTES;
                    const uint32_t bl = al + Cfg::A_BYTES;
#pragma unroll
                    for (int k = 0; k < TC_BK / 16; ++k) {
                        const uint32_t acc_flag = (kb > 0 || k > 0) ? 1u : 0u;
                        const uint32_t koff = k * 32;  // 16 fp16 = 32 bytes along the swizzled row
                        auto mma = [&](uint32_t a, uint32_t b, uint32_t f) {
                            if (CG == 2)
                                tc::mma_f16_pair(d1, tc::smem_desc(a), tc::smem_desc(b), Cfg::IDESC, f);
                            else
                                tc::mma_f16(d1, tc::smem_desc(a), tc::smem_desc(b), Cfg::IDESC, f);
                        };
                        mma(a0 + koff, b0 + koff, acc_flag);
                        if (SPLIT) {
                            if (pr.p.drop_pass != 2) mma(a0 + koff, bl + koff, 1u);
                            if (pr.p.drop_pass != 1) mma(al + koff, b0 + koff, 1u);
                        }
                    }
                    if (CG == 2)  // frees the smem stage (in both CTAs)
                        tc::mma_commit_pair(tc::smem_u32(&bars[S + stage]));
                    else
                        tc::mma_commit(tc::smem_u32(&bars[S + stage]));
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (CG == 2)  // accumulator ready (both CTAs' epilogues)
                    tc::mma_commit_pair(tc::smem_u32(&bars[2 * S + acc]));
                else
                    tc::mma_commit(tc::smem_u32(&bars[2 * S + acc]));
                if (++acc == AS) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else if (warp >= 4) {
        // ------------------------------------------------------------ epilogue
        // 8 warps: warp%4 selects the TMEM lane quarter (hardware access rule),
        // (warp-4)/4 selects which half of the tile's UNITS hidden units.
        const int q = warp & 3;
        const int half = (warp - 4) >> 2;
        constexpr int HU = UNITS / 2;
        float* stg = reinterpret_cast<float*>(smem + S * Cfg::STAGE_BYTES + 256) + (warp - 4) * (CPT ? 512 : 1024);
        int stg_buf = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = cid; t < total_tiles; t += ncl) {
            const int pi = (P.n_prob > 1 && t >= P.prob[1].tile_begin) ? 1 : 0;
            const TcProblem& pr = P.prob[pi];
            const LstmArgs& p = pr.p;
            const int lt = t - pr.tile_begin;
            const int mt = lt / pr.n_tiles, nt = lt - mt * pr.n_tiles;
            const int TRp = tile_rows(p);
            const int row0 = CG == 1 ? mt * TRp : (mt * CG + rank) * TC_BM;  // first row of this CTA's tile
            if (CPT || !p.raw) {
                // cell mode: 16x256b TMEM loads, so the 4 lanes of a quad hold 2 consecutive
                // units each of the same row -- every h / c / split-h store instruction
                // writes whole 32-byte row segments (half the L1 wavefronts of row-per-lane)
                // each instantiation compiles only the epilogues its launches use (fan-out
                // launches run on single CTAs, compacted ones on the CPT instantiation)
                if constexpr (CPT)
                    epilogue_compact<UNITS, SPLIT, CG>(p, Mv, bars, tmem_base, acc, acc_phase, row0, nt, q, half,
                                                       lane, 2 * S, 2 * S + AS, Cfg::ACC_COLS, leader, stg);
                else if (CG == 1 && p.fan > 1)
                    epilogue_fan<UNITS, SPLIT, CG>(p, bars, tmem_base, acc, acc_phase, row0, TRp, nt, q, half, lane,
                                                   2 * S, 2 * S + AS, Cfg::ACC_COLS, leader, pr, stg, stg_buf);
                else
                    epilogue_cells<UNITS, SPLIT, CG>(p, bars, tmem_base, acc, acc_phase, row0, TRp, nt, q, half,
                                                     lane, 2 * S, 2 * S + AS, Cfg::ACC_COLS, leader, pr, stg,
                                                     stg_buf);
                if (++acc == AS) {
                    acc = 0;
                    acc_phase ^= 1;
                }
                continue;
            }
            const int row = row0 + q * 32 + lane;
            const bool valid = row < p.M && (CG == 2 || q * 32 + lane < TRp);
            // raw mode (the context projection P = a_t . W_ctx: no bias, no cell): the
            // pre-activations are stored transposed and split, in the B-operand order of
            // the alpha-block MMA; lane = row, so each 2-byte column store is coalesced
            tc::mbar_wait(tc::smem_u32(&bars[2 * S + acc]), acc_phase);
            tc::fence_after();
            const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * Cfg::ACC_COLS;
            constexpr int NCH = HU / 8;
#pragma unroll 1
            for (int c = 0; c < NCH; ++c) {
                const int uc = half * HU + c * 8;  // unit offset within the tile
                float g[4][8];
#pragma unroll
                for (int gt = 0; gt < 4; ++gt) tc::tmem_ld8(tbase + gt * UNITS + uc, g[gt]);
                tc::tmem_wait_ld();
                if (c == NCH - 1) {  // this warp's TMEM reads are done: release the accumulator
                    tc::fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        if (CG == 2 && !leader)
                            tc::mbar_arrive_remote(tc::smem_u32(&bars[2 * S + AS + acc]), 0);
                        else
                            tc::mbar_arrive(tc::smem_u32(&bars[2 * S + AS + acc]));
                    }
                }
                const float sc = SPLIT ? kSplitUnscale : 1.0f;
                if (SPLIT && pr.tma_out) {
                    // P^T through shared memory: per gate block, the warp's 32 rows x 8
                    // columns of each plane, one bulk tensor store into the [4H][7C] view
                    __half* sp = reinterpret_cast<__half*>(stg);  // [gate][plane][8 n][32 rows]
                    if (lane == 0) tc::bulk_wait_read<0>();      // the previous chunk's stores read it
                    __syncwarp();
#pragma unroll
                    for (int gt = 0; gt < 4; ++gt) {
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            __half hi, lo;
                            split_f16s(g[gt][j] * sc, kPScale, hi, lo);
                            sp[((gt * 2 + 0) * 8 + j) * 32 + lane] = hi;
                            sp[((gt * 2 + 1) * 8 + j) * 32 + lane] = lo;
                        }
                    }
                    tc::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
#pragma unroll
                        for (int gt = 0; gt < 4; ++gt) {
                            const int n0 = nt * Cfg::BN + gt * UNITS + uc;
                            tc::tma_store_2d(&pr.mh, tc::smem_u32(sp + (gt * 2 + 0) * 256), row0 + q * 32, n0);
                            tc::tma_store_2d(&pr.mc, tc::smem_u32(sp + (gt * 2 + 1) * 256), row0 + q * 32, n0);
                        }
                        tc::bulk_commit();
                    }
                    continue;
                }
                if (!valid) continue;
#pragma unroll
                for (int gt = 0; gt < 4; ++gt) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const long long n = (long long)nt * Cfg::BN + gt * UNITS + uc + j;
                        const float v = g[gt][j] * sc;
                        if (SPLIT) {
                            __half hi, lo;
                            split_f16s(v, kPScale, hi, lo);
                            p.pt_hi[n * p.ldt + row] = hi;
                            p.pt_lo[n * p.ldt + row] = lo;
                        } else {
                            reinterpret_cast<__nv_bfloat16*>(p.pt_hi)[n * p.ldt + row] = __float2bfloat16_rn(v);
                        }
                    }
                }
            }
            if (++acc == AS) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
        if (lane == 0) tc::bulk_wait_all();  // this warp's bulk stores are complete
    }
    __syncthreads();
    if (CG == 2) tc::cluster_sync();  // no CTA leaves while its peer may still signal it
    if (warp == 2) {
        tc::fence_after();
        if (CG == 2)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn tc_encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// 2D fp16/bf16 row-major [rows][cols] tensor, box [box_rows][64], 128B swizzle.
bool tc_make_map(CUtensorMap* m, const void* base, long long rows, long long cols, long long row_stride_elems,
              int box_rows) {
    EncodeTiledFn fn = tc_encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)row_stride_elems * 2};
    cuuint32_t box[2] = {(cuuint32_t)TC_BK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, TC_BK == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

namespace {

// fp32 [rows][cols] output view (row stride ld elements), box 32 rows x 8 columns,
// no swizzle: the bulk h / c stores of the cell epilogue
// fan > 1: a 3D [rows][fan][cols] view of the children's rows (child f of parent r is
// row r*fan + f), box 32 parents x 1 child x 8 columns
bool make_out_map(CUtensorMap* m, const float* base, long long rows, int fan, long long cols, long long ld) {
    EncodeTiledFn fn = tc_encode_fn();
    if (!fn || (reinterpret_cast<uintptr_t>(base) & 15) || (ld & 3)) return false;
    CUresult r;
    if (fan <= 1) {
        cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
        cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
        cuuint32_t box[2] = {8, 32};
        cuuint32_t estr[2] = {1, 1};
        r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
        cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)fan, (cuuint64_t)rows};
        cuuint64_t strides[2] = {(cuuint64_t)ld * 4, (cuuint64_t)ld * 4 * fan};
        cuuint32_t box[3] = {8, 1, 32};
        cuuint32_t estr[3] = {1, 1, 1};
        r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    return r == CUDA_SUCCESS;
}

// fp16 [rows][cols] split-h planes (row stride ld elements): box 32 rows x 8 columns
bool make_half_out_map(CUtensorMap* m, const __half* base, long long rows, long long cols, long long ld) {
    EncodeTiledFn fn = tc_encode_fn();
    if (!fn || !base || (reinterpret_cast<uintptr_t>(base) & 15) || (ld & 7)) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
    cuuint32_t box[2] = {8, 32};
    cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// fp16 [n][rows] transposed P planes (row stride ld elements): box 32 rows x 8 n
bool make_pt_out_map(CUtensorMap* m, const __half* base, long long rows, long long n, long long ld) {
    EncodeTiledFn fn = tc_encode_fn();
    if (!fn || !base || (reinterpret_cast<uintptr_t>(base) & 15) || (ld & 7)) return false;
    cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)n};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
    cuuint32_t box[2] = {32, 8};
    cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_map(CUtensorMap* m, const void* base, long long rows, long long cols, long long row_stride_elems,
              int box_rows) {
    return tc_make_map(m, base, rows, cols, row_stride_elems, box_rows);
}

int sm_count() {
    int n = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
}

template <int UNITS, bool SPLIT, int CG>
bool launch_impl(const LstmArgs& a0, const LstmArgs* a1, const __half* Wh0, const __half* Wl0,
                 const __half* Wh1, const __half* Wl1, cudaStream_t stream) {
    using Cfg = TcCfg<UNITS, SPLIT, CG>;
    static std::atomic<unsigned long long> attr{0};
    if (first_on_device(attr)) {
        if (cudaFuncSetAttribute(lstm_gemm_tc<UNITS, SPLIT, CG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 Cfg::SMEM) != cudaSuccess)
            return false;
        if (CG == 1 && cudaFuncSetAttribute(lstm_gemm_tc<UNITS, SPLIT, 1, true>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM) != cudaSuccess)
            return false;
    }
    constexpr int BROWS = Cfg::BN / CG;  // B rows each CTA loads
    TcParams P{};
    CUtensorMap maps[8];
    const LstmArgs* args[2] = {&a0, a1};
    const __half* wh[2] = {Wh0, Wh1};
    const __half* wl[2] = {Wl0, Wl1};
    P.n_prob = a1 ? 2 : 1;
    int tiles = 0;
    for (int i = 0; i < P.n_prob; ++i) {
        const LstmArgs& a = *args[i];
        if (a.K % TC_BK != 0 || a.H % UNITS != 0) return false;
        TcProblem& pr = P.prob[i];
        pr.p = a;
        {
            static const int drop = [] {
                const char* e = std::getenv("KS_F16X2");
                return e ? (e[0] == 'a' ? 1 : e[0] == 'w' ? 2 : 0) : 0;
            }();
            pr.p.drop_pass = drop;
        }
        // the fan-out epilogue writes h, c and the split h of the children (single CTAs)
        if (a.fan > 1 && (a.h_out2 != nullptr || a.raw || CG == 2)) return false;
        // compacted rows: one alpha-block problem on single-CTA 128-row tiles, h / c only
        if (a.cp_M && (a1 || CG == 2 || (a.kb_alpha > 0 && a.alpha_tile != TC_BM) || a.fan > 1 || a.raw ||
                       a.hA_hi || a.h_out2))
            return false;
        {
            static const bool bulk_out = [] {
                const char* e = std::getenv("KS_BULK_OUT");
                return !(e && e[0] == '0');
            }();
            const int fan = a.fan > 1 ? a.fan : 1;
            if (a.raw)  // P^T planes [4H][ldt] fp16: box 32 rows (inner) x 8 gate columns
                pr.tma_out = bulk_out && SPLIT && make_pt_out_map(&pr.mh, a.pt_hi, a.M, 4LL * a.H, a.ldt) &&
                                     make_pt_out_map(&pr.mc, a.pt_lo, a.M, 4LL * a.H, a.ldt)
                                 ? 1
                                 : 0;
            else
                pr.tma_out = bulk_out && !a.cp_M && a.h_out && a.c_out &&
                                     make_out_map(&pr.mh, a.h_out, a.M, fan, a.H, a.ldh) &&
                                     make_out_map(&pr.mc, a.c_out, a.M, fan, a.H, a.ldc)
                                 ? 1
                                 : 0;
            static const bool bulk_a_env = [] {
                const char* e = std::getenv("KS_BULK_A");
                return !(e && e[0] == '0');
            }();
            pr.tma_a = bulk_a_env && pr.tma_out && !a.raw && fan == 1 && SPLIT && a.hA_hi && a.hA_lo && !a.ha_bf16 &&
                               make_half_out_map(&pr.mah, a.hA_hi, a.M, a.H, a.ldha) &&
                               make_half_out_map(&pr.mal, a.hA_lo, a.M, a.H, a.ldha)
                           ? 1
                           : 0;
        }
        if (a.kb_alpha > 0 && (CG == 2 ? a.alpha_tile != 2 * TC_BM : (a.alpha_tile < 1 || a.alpha_tile > TC_BM)))
            return false;  // operand laid out for another tile
        const int tr = (CG == 1 && a.kb_alpha > 0) ? a.alpha_tile : TC_BM;
        pr.m_tiles = ((a.M + tr - 1) / tr + CG - 1) / CG;  // (pair) tiles
        pr.n_tiles = a.H / UNITS;
        pr.k_blocks = a.K / TC_BK;
        pr.tile_begin = tiles;
        tiles += pr.m_tiles * pr.n_tiles;
        // A planes: [M][K] with row stride ldah (default K)
        const long long lda = a.ldah ? a.ldah : a.K;
        if (!make_map(&maps[4 * i + 0], a.A_hi, a.M, a.K, lda, TC_BM)) return false;
        if (!make_map(&maps[4 * i + 1], SPLIT ? a.A_lo : a.A_hi, a.M, a.K, lda, TC_BM)) return false;
        // W planes: the K range after the alpha blocks, at column offset wcol
        const long long ldw = a.ldw ? a.ldw : a.K;
        const long long kw = a.K - (long long)a.kb_alpha * TC_BK;
        const __half* w0 = wh[i] + a.wcol;
        const __half* w1 = (SPLIT ? wl[i] : wh[i]) + a.wcol;
        if (!make_map(&maps[4 * i + 2], w0, 4LL * a.H, kw, ldw, BROWS)) return false;
        if (!make_map(&maps[4 * i + 3], w1, 4LL * a.H, kw, ldw, BROWS)) return false;
    }
    if (P.n_prob == 1) {
        for (int j = 4; j < 8; ++j) maps[j] = maps[j - 4];
        if (a0.kb_alpha > 0) {  // P^T planes in the second problem's B slots
            if (a0.kb_alpha * TC_BK > a0.K) return false;
            if (!make_map(&maps[6], a0.PT_hi, 4LL * a0.H, a0.pt_rows, a0.ldpt, BROWS)) return false;
            if (!make_map(&maps[7], SPLIT ? a0.PT_lo : a0.PT_hi, 4LL * a0.H, a0.pt_rows, a0.ldpt, BROWS))
                return false;
        }
    } else if (a0.kb_alpha > 0 || (a1 && a1->kb_alpha > 0)) {
        return false;
    }
    P.total_tiles = tiles;
    const int units = sm_count() / CG;  // persistent: one CTA (pair) per SM (pair)
    const int grid = CG * (tiles < units ? tiles : units);
    if (CG == 1) {
        if (a0.cp_M)
            lstm_gemm_tc<UNITS, SPLIT, 1, true><<<grid, 640, Cfg::SMEM, stream>>>(
                P, maps[0], maps[1], maps[2], maps[3], maps[4], maps[5], maps[6], maps[7]);
        else
            lstm_gemm_tc<UNITS, SPLIT, CG><<<grid, 384, Cfg::SMEM, stream>>>(P, maps[0], maps[1], maps[2], maps[3],
                                                                              maps[4], maps[5], maps[6], maps[7]);
        return cudaGetLastError() == cudaSuccess;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(384);
    cfg.dynamicSmemBytes = Cfg::SMEM;
    cfg.stream = stream;
    cudaLaunchAttribute attr_c[1];
    attr_c[0].id = cudaLaunchAttributeClusterDimension;
    attr_c[0].val.clusterDim.x = 2;
    attr_c[0].val.clusterDim.y = 1;
    attr_c[0].val.clusterDim.z = 1;
    cfg.attrs = attr_c;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, lstm_gemm_tc<UNITS, SPLIT, CG>, P, maps[0], maps[1], maps[2], maps[3], maps[4],
                              maps[5], maps[6], maps[7]) == cudaSuccess;
}

}  // namespace

int tc_units_default() { return 32; }

bool launch_lstm_tc(const LstmArgs& a0, const LstmArgs* a1, int mode, const __half* W_hi0,
                    const __half* W_lo0, const __half* W_hi1, const __half* W_lo1, cudaStream_t stream,
                    int* launches, int units, bool pair) {
    bool ok;
    if (pair && units == 64)
        ok = mode == 0 ? launch_impl<64, true, 2>(a0, a1, W_hi0, W_lo0, W_hi1, W_lo1, stream)
                       : launch_impl<64, false, 2>(a0, a1, W_hi0, W_lo0, W_hi1, W_lo1, stream);
    else if (mode == 0)
        ok = units == 64 ? launch_impl<64, true, 1>(a0, a1, W_hi0, W_lo0, W_hi1, W_lo1, stream)
                         : launch_impl<32, true, 1>(a0, a1, W_hi0, W_lo0, W_hi1, W_lo1, stream);
    else
        ok = units == 64 ? launch_impl<64, false, 1>(a0, a1, W_hi0, W_lo0, W_hi1, W_lo1, stream)
                         : launch_impl<32, false, 1>(a0, a1, W_hi0, W_lo0, W_hi1, W_lo1, stream);
    if (ok && launches) *launches = 1;
    return ok;
}

}  // namespace ksb
