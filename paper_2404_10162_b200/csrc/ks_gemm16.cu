// ks_gemm16.cu -- the training contractions on the 5th-generation tensor cores.
//
//   C[M x N] = 2^-(eA+eB) * (A_hi.B_hi + A_hi.B_lo + A_lo.B_hi)  (+ beta * C)
//
// F16X3 operand planes: x 2^e = hi + lo, both fp16, at a per-operand power-of-two
// scale chosen from max |x| (ks_train.cu k_split_planes), ~22-bit operands; the
// three products accumulate in one fp32 TMEM accumulator -- the fp32-grade
// product the reference's fp64 training body (models.cpp:905-947,
// autodiff.cpp:326-544) needs.  The planes keep their source's row-major layout
// and each operand is read K-major or MN-major as the contraction needs
// (instruction-descriptor a_major / b_major), so one split of a matrix serves
// every GEMM it appears in, transposed or not: W in the forward (B, MN-major)
// and in dX (B^T, K-major); the activations X in the forward (A, K-major) and in
// dW = X^T dZ (A, MN-major); dZ in dX (A, K-major) and in dW (B, MN-major).
// The scale exponents are read from the operands' max|x| slots on the device,
// so a captured CUDA graph replays them.
//
// Structure (the decode GEMM's, ks_gemm_tc.cu, with a plain-store epilogue):
// persistent CTAs, 384 threads --
//   warp 0      TMA producer (hi and lo boxes of A and B, 128B swizzle, mbarrier ring)
//   warp 1      MMA issuer (one thread, 3 x tcgen05.mma.cta_group::1.kind::f16 per K=16)
//   warp 2      TMEM allocator (2 accumulators x BN fp32 columns)
//   warps 4..11 epilogue: tcgen05.ld -> alpha, beta -> fp32 stores
// Shared-memory operand layouts (SWIZZLE_128B): K-major tiles are rows of 64 K
// (one box [rows][64]); MN-major tiles are boxes of [64 K rows][64 MN] (8 KB,
// one per 64 MN), canonical ((8,n),(8,k)):((1,LBO),(8,SBO)) in 16-byte units:
// LBO = 8 KB between MN boxes, SBO = 1 KB between 8-row K groups, and a K=16
// step advances 2 KB.
// Work item = (128-row tile, BN-column tile, K split).  Long reductions with few
// output tiles (the weight gradients: K = T x batch) are split along K when that
// shortens the makespan; split partials go to a workspace and a fixed-order
// reduction (deterministic) applies alpha / beta.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>

#include "ks_common.cuh"
#include "ks_tc.cuh"

namespace ksb {

namespace {

constexpr int G_BM = 128;
constexpr int G_BK = kTcBK;  // 64 fp16 = one 128-byte swizzled row

template <int BN, int CG>
struct GCfg {
    static constexpr int A_BYTES = G_BM * G_BK * 2;        // one plane
    static constexpr int B_BYTES = (BN / CG) * G_BK * 2;   // this CTA's share (CTA pair: half the N rows)
    static constexpr int STAGE_BYTES = 2 * (A_BYTES + B_BYTES);
    static constexpr int STAGES = (200 * 1024) / STAGE_BYTES > 6 ? 6 : (200 * 1024) / STAGE_BYTES;
    static constexpr int ACC_COLS = BN;
    static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
};
// fp32 accumulate, fp16 A/B, a_major (bit 15) / b_major (bit 16): 1 = MN-major,
// N >> 3 at bits 17-22, M >> 4 at bits 24-28
template <int BN, bool AMN, bool BMN, int CG>
constexpr uint32_t g_idesc() {
    return (1u << 4) | ((AMN ? 1u : 0u) << 15) | ((BMN ? 1u : 0u) << 16) | ((uint32_t)(BN >> 3) << 17) |
           ((uint32_t)((CG * G_BM) >> 4) << 24);
}
// MN-major SW128 descriptor: LBO = 8 KB (next 64 MN), SBO = 1 KB (next 8 K rows)
__device__ __forceinline__ uint64_t desc_mn(uint32_t addr) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)(8192 >> 4) << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

struct GParams {
    int M, N;
    int m_tiles, n_tiles, k_blocks, splits, kb_per_split;
    int total;                // m_tiles * n_tiles * splits
    float* C;
    long long ldc;
    const int* amaxA;         // device max|x| slots -> scale exponents
    const int* amaxB;
    const float* beta;        // device scalar, null: 0
    float* part;              // [splits][M][N] when splits > 1
};

// CG = 2: a CTA pair (cluster of 2) runs M = 256 tcgen05.mma.cta_group::2 tiles, each
// CTA holding its 128 A rows and half of the B tile (as the decode GEMM's pair mode)
template <int BN, bool AMN, bool BMN, int CG>
__global__ void __launch_bounds__(384, 1)
    gemm16_tc(const __grid_constant__ GParams P, const __grid_constant__ CUtensorMap mAh,
              const __grid_constant__ CUtensorMap mAl, const __grid_constant__ CUtensorMap mBh,
              const __grid_constant__ CUtensorMap mBl) {
    using Cfg = GCfg<BN, CG>;
    constexpr int S = Cfg::STAGES;
    constexpr uint32_t IDESC = g_idesc<BN, AMN, BMN, CG>();
    const int rank = CG == 2 ? (int)tc::cluster_rank() : 0;
    const bool leader = rank == 0;
    const int cid = blockIdx.x / CG, ncl = gridDim.x / CG;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * Cfg::STAGE_BYTES);
    // full[S], empty[S], tfull[2], tempty[2], TMEM base slot
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 4);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            tc::mbar_init(tc::smem_u32(&bars[s]), 1);
            tc::mbar_init(tc::smem_u32(&bars[S + s]), 1);
        }
        for (int a = 0; a < 2; ++a) {
            tc::mbar_init(tc::smem_u32(&bars[2 * S + a]), 1);
            tc::mbar_init(tc::smem_u32(&bars[2 * S + 2 + a]), 8 * CG);  // one arrive per epilogue warp (of the pair)
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        tc::tma_prefetch(&mAh);
        tc::tma_prefetch(&mAl);
        tc::tma_prefetch(&mBh);
        tc::tma_prefetch(&mBl);
    }
    if (warp == 2) {
        if (CG == 2) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             tc::smem_u32(tmem_slot)), "n"(2 * BN)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             tc::smem_u32(tmem_slot)), "n"(2 * BN)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
    }
    tc::fence_before();
    __syncthreads();
    if (CG == 2) tc::cluster_sync();  // the peer's barriers are initialised before any remote arrive
    tc::fence_after();
    const uint32_t tmem_base = *tmem_slot;

    auto work = [&](int w, int& mt, int& nt, int& kb0, int& kb1) {
        const int sp = w % P.splits, tile = w / P.splits;
        mt = tile / P.n_tiles;
        nt = tile - mt * P.n_tiles;
        kb0 = sp * P.kb_per_split;
        kb1 = min(P.k_blocks, kb0 + P.kb_per_split);
    };

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            auto load = [&](uint32_t dst, const CUtensorMap* m, uint32_t bar, int x, int y) {
                if (CG == 2)
                    tc::tma_load_2d_pair(dst, m, bar, x, y);  // completes on the leader's barrier
                else
                    tc::tma_load_2d(dst, m, bar, x, y);
            };
            for (int w = cid; w < P.total; w += ncl) {
                int mt, nt, kb0, kb1;
                work(w, mt, nt, kb0, kb1);
                const int arow = (mt * CG + rank) * G_BM;         // this CTA's A rows
                const int bn0 = nt * BN + rank * (BN / CG);      // this CTA's B rows / columns
                for (int kb = kb0; kb < kb1; ++kb) {
                    tc::mbar_wait(tc::smem_u32(&bars[S + stage]), phase ^ 1);
                    const uint32_t full = tc::smem_u32(&bars[stage]);
                    if (leader) tc::mbar_expect_tx(full, CG * Cfg::STAGE_BYTES);  // both CTAs' bytes
                    const uint32_t st = tc::smem_u32(smem + stage * Cfg::STAGE_BYTES);
                    // stage: A_hi | A_lo | B_hi | B_lo
#pragma unroll
                    for (int pl = 0; pl < 2; ++pl) {
                        const uint32_t da = st + pl * Cfg::A_BYTES;
                        const CUtensorMap* ma = pl ? &mAl : &mAh;
                        if (AMN) {
#pragma unroll
                            for (int j = 0; j < G_BM / 64; ++j) load(da + j * 8192, ma, full, arow + j * 64, kb * G_BK);
                        } else {
                            load(da, ma, full, kb * G_BK, arow);
                        }
                        const uint32_t db = st + 2 * Cfg::A_BYTES + pl * Cfg::B_BYTES;
                        const CUtensorMap* mb = pl ? &mBl : &mBh;
                        if (BMN) {
#pragma unroll
                            for (int j = 0; j < BN / CG / 64; ++j) load(db + j * 8192, mb, full, bn0 + j * 64, kb * G_BK);
                        } else {
                            load(db, mb, full, kb * G_BK, bn0);
                        }
                    }
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && leader) {
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0;
            auto mma = [&](uint32_t d, uint64_t a, uint64_t b, uint32_t f) {
                if (CG == 2)
                    tc::mma_f16_pair(d, a, b, IDESC, f);
                else
                    tc::mma_f16(d, a, b, IDESC, f);
            };
            auto commit = [&](uint32_t bar) {
                if (CG == 2)
                    tc::mma_commit_pair(bar);  // arrives on the barrier in both CTAs
                else
                    tc::mma_commit(bar);
            };
            for (int w = cid; w < P.total; w += ncl) {
                int mt, nt, kb0, kb1;
                work(w, mt, nt, kb0, kb1);
                tc::mbar_wait(tc::smem_u32(&bars[2 * S + 2 + acc]), acc_phase ^ 1);
                tc::fence_after();
                const uint32_t d = tmem_base + acc * Cfg::ACC_COLS;
                for (int kb = kb0; kb < kb1; ++kb) {
                    tc::mbar_wait(tc::smem_u32(&bars[stage]), phase);
                    tc::fence_after();
                    const uint32_t ah = tc::smem_u32(smem + stage * Cfg::STAGE_BYTES);
                    const uint32_t al = ah + Cfg::A_BYTES;
                    const uint32_t bh = al + Cfg::A_BYTES;
                    const uint32_t bl = bh + Cfg::B_BYTES;
#pragma unroll
                    for (int k = 0; k < G_BK / 16; ++k) {
                        // K = 16: 32 bytes along a K-major row, or 16 rows (2 KB) of an MN-major box
                        auto da = [&](uint32_t a) { return AMN ? desc_mn(a + k * 2048) : tc::smem_desc(a + k * 32); };
                        auto db = [&](uint32_t b) { return BMN ? desc_mn(b + k * 2048) : tc::smem_desc(b + k * 32); };
                        mma(d, da(ah), db(bh), (kb > kb0 || k > 0) ? 1u : 0u);
                        mma(d, da(ah), db(bl), 1u);
                        mma(d, da(al), db(bh), 1u);
                    }
                    commit(tc::smem_u32(&bars[S + stage]));
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                commit(tc::smem_u32(&bars[2 * S + acc]));
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else if (warp >= 4) {
        // warp % 4: TMEM lane quarter (rows q*32 .. q*32+31); (warp - 4) / 4: column half
        const int q = warp & 3, half = (warp - 4) >> 2;
        constexpr int HC = BN / 2;
        const float alpha = exp2f(-(float)(f16_scale_exp(*P.amaxA) + f16_scale_exp(*P.amaxB)));
        const float beta = P.beta ? *P.beta : 0.0f;
        const bool vec = (P.ldc & 3) == 0 && (reinterpret_cast<uintptr_t>(P.C) & 15) == 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int w = cid; w < P.total; w += ncl) {
            int mt, nt, kb0, kb1;
            work(w, mt, nt, kb0, kb1);
            const int sp = w % P.splits;
            const int row = (mt * CG + rank) * G_BM + q * 32 + lane;
            tc::mbar_wait(tc::smem_u32(&bars[2 * S + acc]), acc_phase);
            tc::fence_after();
            const uint32_t tb = tmem_base + ((uint32_t)(q * 32) << 16) + acc * Cfg::ACC_COLS + half * HC;
#pragma unroll 1
            for (int c = 0; c < HC; c += 16) {
                float v[16];
                tc::tmem_ld8(tb + c, v);
                tc::tmem_ld8(tb + c + 8, v + 8);
                tc::tmem_wait_ld();
                if (c + 16 >= HC) {  // this warp's reads of the accumulator are done
                    tc::fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        if (CG == 2 && !leader)
                            tc::mbar_arrive_remote(tc::smem_u32(&bars[2 * S + 2 + acc]), 0);
                        else
                            tc::mbar_arrive(tc::smem_u32(&bars[2 * S + 2 + acc]));
                    }
                }
                const int col = nt * BN + half * HC + c;
                if (row >= P.M || col >= P.N) continue;
                if (P.splits > 1) {
                    float* dst = P.part + ((long long)sp * P.M + row) * P.N + col;
                    if (col + 16 <= P.N && (P.N & 3) == 0) {
#pragma unroll
                        for (int j = 0; j < 16; j += 4)
                            *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                    } else {
#pragma unroll
                        for (int j = 0; j < 16; ++j)
                            if (col + j < P.N) dst[j] = v[j];
                    }
                    continue;
                }
                float* dst = P.C + (long long)row * P.ldc + col;
                if (col + 16 <= P.N && vec) {
#pragma unroll
                    for (int j = 0; j < 16; j += 4) {
                        float4 o = make_float4(alpha * v[j], alpha * v[j + 1], alpha * v[j + 2], alpha * v[j + 3]);
                        if (beta != 0.0f) {
                            const float4 cv = *reinterpret_cast<const float4*>(dst + j);
                            o.x = fmaf(beta, cv.x, o.x);
                            o.y = fmaf(beta, cv.y, o.y);
                            o.z = fmaf(beta, cv.z, o.z);
                            o.w = fmaf(beta, cv.w, o.w);
                        }
                        *reinterpret_cast<float4*>(dst + j) = o;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        if (col + j >= P.N) break;
                        float o = alpha * v[j];
                        if (beta != 0.0f) o = fmaf(beta, dst[j], o);
                        dst[j] = o;
                    }
                }
            }
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    }
    __syncthreads();
    if (CG == 2) tc::cluster_sync();  // no CTA leaves while its peer may still signal it
    if (warp == 2) {
        tc::fence_after();
        if (CG == 2)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(2 * BN)
                         : "memory");
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(2 * BN)
                         : "memory");
    }
}

// C = alpha * sum_s part[s] + beta * C, s ascending (fixed order); 4 columns per thread
__global__ void gemm16_reduce(const float* part, int splits, int M, int N, float* C, long long ldc,
                              const int* amaxA, const int* amaxB, const float* beta_p) {
    const float alpha = exp2f(-(float)(f16_scale_exp(*amaxA) + f16_scale_exp(*amaxB)));
    const float beta = beta_p ? *beta_p : 0.0f;
    const long long plane = (long long)M * N;
    const int nq = (N + 3) / 4;
    const long long n = (long long)M * nq;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / nq;
        const int c0 = (int)(i - r * nq) * 4;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int c = c0 + j;
            if (c >= N) break;
            const long long e = r * N + c;
            float s = part[e];
            for (int k = 1; k < splits; ++k) s += part[k * plane + e];
            float* dst = C + r * ldc + c;
            float o = alpha * s;
            if (beta != 0.0f) o = fmaf(beta, *dst, o);
            *dst = o;
        }
    }
}

template <int BN, bool AMN, bool BMN, int CG>
bool launch_t(const GemmF16Args& g, int splits, cudaStream_t stream) {
    using Cfg = GCfg<BN, CG>;
    static std::atomic<unsigned long long> attr{0};
    if (first_on_device(attr) && cudaFuncSetAttribute(gemm16_tc<BN, AMN, BMN, CG>,
                                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                      Cfg::SMEM) != cudaSuccess)
        return false;
    // K-major planes: [rows = M|N][cols = K], box [rows][64];  MN-major: [rows = K][cols = M|N],
    // box [64][64].  A CTA pair loads half of each B tile per CTA.
    CUtensorMap m[4];
    for (int pl = 0; pl < 2; ++pl) {
        const __half* a = pl ? g.A_lo : g.A_hi;
        const __half* b = pl ? g.B_lo : g.B_hi;
        const bool oka = AMN ? tc_make_map(&m[pl], a, g.K, g.M, g.lda, 64) : tc_make_map(&m[pl], a, g.M, g.K, g.lda, G_BM);
        const bool okb = BMN ? tc_make_map(&m[2 + pl], b, g.K, g.N, g.ldb, 64)
                             : tc_make_map(&m[2 + pl], b, g.N, g.K, g.ldb, BN / CG);
        if (!oka || !okb) return false;
    }
    GParams P{};
    P.M = g.M;
    P.N = g.N;
    P.m_tiles = (g.M + CG * G_BM - 1) / (CG * G_BM);
    P.n_tiles = (g.N + BN - 1) / BN;
    P.k_blocks = (int)((g.K + G_BK - 1) / G_BK);
    P.kb_per_split = (P.k_blocks + splits - 1) / splits;
    P.splits = (P.k_blocks + P.kb_per_split - 1) / P.kb_per_split;  // every split non-empty
    P.total = P.m_tiles * P.n_tiles * P.splits;
    P.C = g.C;
    P.ldc = g.ldc;
    P.amaxA = g.amaxA;
    P.amaxB = g.amaxB;
    P.beta = g.beta;
    P.part = g.part;
    const int grid = CG * std::min(P.total, g.sms / CG);
    if (CG == 1) {
        gemm16_tc<BN, AMN, BMN, CG><<<grid, 384, Cfg::SMEM, stream>>>(P, m[0], m[1], m[2], m[3]);
        if (cudaGetLastError() != cudaSuccess) return false;
    } else {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((unsigned)grid);
        cfg.blockDim = dim3(384);
        cfg.dynamicSmemBytes = Cfg::SMEM;
        cfg.stream = stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        if (cudaLaunchKernelEx(&cfg, gemm16_tc<BN, AMN, BMN, CG>, P, m[0], m[1], m[2], m[3]) != cudaSuccess)
            return false;
    }
    if (P.splits > 1) {
        const long long n = (long long)g.M * ((g.N + 3) / 4);
        const int blocks = (int)std::min<long long>((n + 255) / 256, 8LL * g.sms);
        gemm16_reduce<<<blocks, 256, 0, stream>>>(g.part, P.splits, g.M, g.N, g.C, g.ldc, g.amaxA, g.amaxB, g.beta);
        if (cudaGetLastError() != cudaSuccess) return false;
    }
    return true;
}

template <int BN, int CG>
bool launch_bn(const GemmF16Args& g, int splits, cudaStream_t stream) {
    if (g.a_mn)
        return g.b_mn ? launch_t<BN, true, true, CG>(g, splits, stream) : launch_t<BN, true, false, CG>(g, splits, stream);
    return g.b_mn ? launch_t<BN, false, true, CG>(g, splits, stream) : launch_t<BN, false, false, CG>(g, splits, stream);
}

}  // namespace

namespace {
// modelled time of a (BN, CTA group, splits) choice: the tensor-core makespan (waves
// of work items over the SMs / CTA pairs; a full-K 128 x BN tile = 3 x 2 x 128 x BN x
// K FLOP at ~9 TFLOP/s per SM, BN = 128 tiles ~10% slower per FLOP: A is re-staged
// per N tile; a CTA pair runs a 256-row tile in the time of a 128-row one at ~15%
// higher issue rate: half the B operand traffic per SM) plus, when split, the
// reduction pass ((splits + 2) x M x N x 4 bytes at ~2.5 TB/s, plus a launch)
double gemm16_cost(int M, int N, long long K, int sms, int bn, int cg, int s) {
    const long long tiles = (long long)((M + cg * G_BM - 1) / (cg * G_BM)) * ((N + bn - 1) / bn);
    const double tile_s = 6.0 * G_BM * bn * (double)K / 9.0e12 * (bn == 128 ? 1.1 : 1.0) * (cg == 2 ? 0.87 : 1.0);
    const long long slots = sms / cg;
    double c = (double)((tiles * s + slots - 1) / slots) * tile_s / (double)s;
    if (s > 1) c += (s + 2.0) * (double)M * N * 4.0 / 2.5e12 + 5e-6;
    return c;
}
void gemm16_plan(int M, int N, long long K, int sms, int& bn, int& cg, int& splits) {
    static const bool pairs = [] {
        const char* e = std::getenv("KS_TRAIN_PAIR");
        return !(e && e[0] == '0');
    }();
    const long long kb = (K + G_BK - 1) / G_BK;
    bn = N <= 128 ? 128 : 256;
    cg = 1;
    splits = 1;
    double best = gemm16_cost(M, N, K, sms, bn, 1, 1);
    for (int c2 : {1, 2}) {
        if (c2 == 2 && (!pairs || M <= G_BM)) continue;
        for (int b : {128, 256}) {
            if (b == 256 && N <= 128) continue;
            for (long long s = 1; s <= 64 && (s == 1 || s * 4 <= kb); ++s) {
                const double c = gemm16_cost(M, N, K, sms, b, c2, (int)s);
                if (c < best * 0.999) {
                    best = c;
                    bn = b;
                    cg = c2;
                    splits = (int)s;
                }
            }
        }
    }
}
}  // namespace

int gemm16_splits(int M, int N, long long K, int sms) {
    int bn, cg, s;
    gemm16_plan(M, N, K, sms, bn, cg, s);
    return s;
}

bool launch_gemm16(const GemmF16Args& g, cudaStream_t stream, int* launches) {
    if (g.M <= 0 || g.N <= 0 || g.K <= 0) return false;
    if ((g.lda % 8) != 0 || (g.ldb % 8) != 0) return false;  // TMA: 16-byte row strides
    int bn, cg, splits;
    gemm16_plan(g.M, g.N, g.K, g.sms, bn, cg, splits);
    if (splits > 1 && g.part == nullptr) return false;
    bool ok;
    if (cg == 2)
        ok = bn == 128 ? launch_bn<128, 2>(g, splits, stream) : launch_bn<256, 2>(g, splits, stream);
    else
        ok = bn == 128 ? launch_bn<128, 1>(g, splits, stream) : launch_bn<256, 1>(g, splits, stream);
    if (ok && launches) *launches += splits > 1 ? 2 : 1;
    return ok;
}

// ---------------------------------------------------------------------------
// F16X3 operand planes
// ---------------------------------------------------------------------------
namespace {

// F16X3 operand split (ksb::f16_scale_exp, ks_tc.cuh): x 2^e = hi + lo with hi,
// lo fp16 (~22-bit operands, like the decode GEMM's F16X3); e from the operand's
// max |x| so that |x| 2^e < 2^14; entries above 2^-28 max|x| keep full relative
// precision.  hi.hi + hi.lo + lo.hi (the tcgen05 GEMM, ks_gemm16.cu) times
// 2^-(eA+eB) recovers an fp32-grade product at the fp16 tensor-core rate.
// max |x| of a row-major block into *out (pre-zeroed; non-negative floats order as ints)
__global__ void __launch_bounds__(256) k_absmax(const float* src, long long rows, long long cols, long long ld, int* out) {
    __shared__ float wm[8];
    float m = 0.0f;
    for (long long r = blockIdx.y; r < rows; r += gridDim.y)
        for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < cols; c += (long long)gridDim.x * blockDim.x)
            m = fmaxf(m, fabsf(src[r * ld + c]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {  // one atomic per block
        m = threadIdx.x < (blockDim.x >> 5) ? wm[threadIdx.x] : 0.0f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (threadIdx.x == 0 && m > 0.0f) atomicMax(out, __float_as_int(m));
    }
}
__device__ __forceinline__ void split_f16x2s(float x, float y, float sc, __half2& hi, __half2& lo) {
    const float2 v = __fmul2_rn(make_float2(x, y), make_float2(sc, sc));
    hi = __float22half2_rn(v);
    const float2 h = __half22float2(hi);
    lo = __float22half2_rn(__fadd2_rn(v, make_float2(-h.x, -h.y)));
}
// hi / lo planes of a row-major block, same layout (row stride ldo), 4 columns per
// thread when aligned; flat grid-stride over (row, column group)
__global__ void k_split_planes(const float* src, long long rows, int cols, long long ld, __half* hi, __half* lo,
                               long long ldo, const int* amax) {
    const float sc = exp2f((float)f16_scale_exp(*amax));
    const bool vec = (cols & 3) == 0 && (ld & 3) == 0 && (ldo & 3) == 0 &&
                     ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(hi) |
                       reinterpret_cast<uintptr_t>(lo)) & 15) == 0;
    const int cw = vec ? cols >> 2 : cols;
    const long long n = rows * (long long)cw;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / cw;
        const int c = (int)(i - r * cw);
        if (vec) {
            const float4 x = reinterpret_cast<const float4*>(src + r * ld)[c];
            __half2 h01, l01, h23, l23;
            split_f16x2s(x.x, x.y, sc, h01, l01);
            split_f16x2s(x.z, x.w, sc, h23, l23);
            uint2 hv, lv;
            hv.x = *reinterpret_cast<uint32_t*>(&h01);
            hv.y = *reinterpret_cast<uint32_t*>(&h23);
            lv.x = *reinterpret_cast<uint32_t*>(&l01);
            lv.y = *reinterpret_cast<uint32_t*>(&l23);
            reinterpret_cast<uint2*>(hi + r * ldo)[c] = hv;
            reinterpret_cast<uint2*>(lo + r * ldo)[c] = lv;
        } else {
            const float x = src[r * ld + c] * sc;
            const __half h = __float2half_rn(x);
            hi[r * ldo + c] = h;
            lo[r * ldo + c] = __float2half_rn(x - __half2float(h));
        }
    }
}

}  // namespace

void launch_absmax(const float* src, long long rows, long long cols, long long ld, int* out, cudaStream_t s) {
    const unsigned gx = (unsigned)std::min<long long>((cols + 255) / 256, 8);
    dim3 grid(gx, (unsigned)std::min<long long>(rows, std::max<long long>(1, 1184 / gx)));
    k_absmax<<<grid, 256, 0, s>>>(src, rows, cols, ld, out);
}

void launch_split_planes(const float* src, long long rows, long long cols, long long ld, __half* hi, __half* lo,
                         long long ldo, const int* amax, cudaStream_t s) {
    const long long items = rows * ((cols + 3) / 4);
    const unsigned grid = (unsigned)std::max<long long>(1, std::min<long long>((items + 255) / 256, 148LL * 16));
    k_split_planes<<<grid, 256, 0, s>>>(src, rows, (int)cols, ld, hi, lo, ldo, amax);
}

// ---------------------------------------------------------------------------
// fp32 SIMT GEMM (exact fp32 FMA, any transposes): the narrow training
// contractions (heads, attention: an output side below 16 columns, where a
// 128 x 128+ tensor-core tile would be mostly padding) and KS_TRAIN_GEMM=fp32.
//   C[M x N] = op(A) op(B) + beta C, row-major; op(A)[m][k] = ta ? A[k][m] : A[m][k]
// 64 x 64 output tile per 256-thread CTA (4 x 4 per thread), K slabs of 16 in
// shared memory; short output / long reduction shapes split K over grid.z
// into a workspace reduced in fixed order.
namespace {

constexpr int SG_BM = 64, SG_BN = 64, SG_BK = 16;

struct SgArgs {
    int M, N;
    long long K;
    const float* A;
    long long lda;
    const float* B;
    long long ldb;
    int ta, tb;
    float beta;
    float* C;
    long long ldc;
    float* part;
    long long kchunk;
};

__global__ void __launch_bounds__(256) sgemm_tile(const SgArgs a) {
    __shared__ float As[SG_BK][SG_BM + 4];
    __shared__ float Bs[SG_BK][SG_BN + 4];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int m0 = blockIdx.y * SG_BM, n0 = blockIdx.x * SG_BN;
    const long long k0 = (long long)blockIdx.z * a.kchunk;
    const long long k1 = min(a.K, k0 + a.kchunk);
    float acc[4][4] = {};
    for (long long kk = k0; kk < k1; kk += SG_BK) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int i = tid + j * 256;  // 0..1023
            // A slab: 64 (m) x 16 (k); consecutive threads walk the contiguous dimension
            int mm, kq;
            if (a.ta) { mm = i & 63; kq = i >> 6; } else { kq = i & 15; mm = i >> 4; }
            const long long gk = kk + kq;
            const int gm = m0 + mm;
            float v = 0.0f;
            if (gk < k1 && gm < a.M) v = a.ta ? a.A[gk * a.lda + gm] : a.A[(long long)gm * a.lda + gk];
            As[kq][mm] = v;
            int nn, kb;
            if (a.tb) { kb = i & 15; nn = i >> 4; } else { nn = i & 63; kb = i >> 6; }
            const long long gkb = kk + kb;
            const int gn = n0 + nn;
            float w = 0.0f;
            if (gkb < k1 && gn < a.N) w = a.tb ? a.B[(long long)gn * a.ldb + gkb] : a.B[gkb * a.ldb + gn];
            Bs[kb][nn] = w;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < SG_BK; ++k) {
            float av[4], bv[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) av[r] = As[k][ty * 4 + r];
#pragma unroll
            for (int c = 0; c < 4; ++c) bv[c] = Bs[k][tx * 4 + c];
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[r][c] = fmaf(av[r], bv[c], acc[r][c]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int m = m0 + ty * 4 + r;
        if (m >= a.M) continue;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int n = n0 + tx * 4 + c;
            if (n >= a.N) continue;
            if (a.part) {
                a.part[((long long)blockIdx.z * a.M + m) * a.N + n] = acc[r][c];
            } else {
                float* d = a.C + (long long)m * a.ldc + n;
                *d = a.beta != 0.0f ? fmaf(a.beta, *d, acc[r][c]) : acc[r][c];
            }
        }
    }
}

// many splits, few outputs: one warp per output, lanes over the splits (fixed-order shuffle tree)
__global__ void sgemm_reduce_warp(const float* part, int splits, int M, int N, float* C, long long ldc, float beta) {
    const long long n = (long long)M * N;
    const long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    float s = 0.0f;
    for (int k = lane; k < splits; k += 32) s += part[k * n + i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
        const long long r = i / N, c = i - r * N;
        float* d = C + r * ldc + c;
        *d = beta != 0.0f ? fmaf(beta, *d, s) : s;
    }
}
__global__ void sgemm_reduce(const float* part, int splits, int M, int N, float* C, long long ldc, float beta) {
    const long long n = (long long)M * N;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        float s = part[i];
        for (int k = 1; k < splits; ++k) s += part[k * n + i];
        const long long r = i / N, c = i - r * N;
        float* d = C + r * ldc + c;
        *d = beta != 0.0f ? fmaf(beta, *d, s) : s;
    }
}

// Narrow outputs (N <= 16: heads, attention scores / weights).
//  rows:  op(A) = A (M x K rows): one warp per output row, lanes over K, the N
//         partial sums reduced by shuffles (fixed order).
//  cols:  op(A) = A^T (A stored K x M): one thread per output row m (coalesced
//         along m), a K chunk per grid.y, partials reduced in fixed order.
template <int NN>
__global__ void __launch_bounds__(256) sgemm_narrow_rows(const SgArgs a) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int m = warp; m < a.M; m += nw) {
        float acc[NN];
#pragma unroll
        for (int n = 0; n < NN; ++n) acc[n] = 0.0f;
        const float* ar = a.A + (long long)m * a.lda;
        for (long long k = lane; k < a.K; k += 32) {
            const float x = ar[k];
#pragma unroll
            for (int n = 0; n < NN; ++n)
                if (n < a.N) acc[n] = fmaf(x, a.tb ? a.B[(long long)n * a.ldb + k] : a.B[k * a.ldb + n], acc[n]);
        }
#pragma unroll
        for (int n = 0; n < NN; ++n) {
            float v = acc[n];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            acc[n] = v;
        }
        if (lane < a.N) {
            float v = acc[0];
#pragma unroll
            for (int n = 1; n < NN; ++n)
                if (n == lane) v = acc[n];
            float* d = a.C + (long long)m * a.ldc + lane;
            *d = a.beta != 0.0f ? fmaf(a.beta, *d, v) : v;
        }
    }
}
template <int NN>
__global__ void __launch_bounds__(256) sgemm_narrow_cols(const SgArgs a) {
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    const long long k0 = (long long)blockIdx.y * a.kchunk;
    const long long k1 = min(a.K, k0 + a.kchunk);
    __shared__ float bs[64][NN];
    float acc[NN];
#pragma unroll
    for (int n = 0; n < NN; ++n) acc[n] = 0.0f;
    for (long long kk = k0; kk < k1; kk += 64) {
        __syncthreads();
        for (int i = threadIdx.x; i < 64 * NN; i += blockDim.x) {
            const int kq = i / NN, n = i - kq * NN;
            const long long k = kk + kq;
            bs[kq][n] = (k < k1 && n < a.N) ? (a.tb ? a.B[(long long)n * a.ldb + k] : a.B[k * a.ldb + n]) : 0.0f;
        }
        __syncthreads();
        if (m < a.M) {
            const int kn = (int)min(64LL, k1 - kk);
            for (int kq = 0; kq < kn; ++kq) {
                const float x = a.A[(kk + kq) * a.lda + m];
#pragma unroll
                for (int n = 0; n < NN; ++n) acc[n] = fmaf(x, bs[kq][n], acc[n]);
            }
        }
    }
    if (m >= a.M) return;
#pragma unroll
    for (int n = 0; n < NN; ++n) {
        if (n >= a.N) break;
        if (a.part) {
            a.part[((long long)blockIdx.y * a.M + m) * a.N + n] = acc[n];
        } else {
            float* d = a.C + (long long)m * a.ldc + n;
            *d = a.beta != 0.0f ? fmaf(a.beta, *d, acc[n]) : acc[n];
        }
    }
}

// K chunk of the narrow column kernel: enough (row block, chunk) CTAs for ~2 waves
long long narrow_kchunk(int M, long long K, int sms) {
    const long long rb = (M + 255) / 256;
    long long chunks = std::max(1LL, std::min((4LL * sms + rb - 1) / rb, (K + 63) / 64));
    chunks = std::min(chunks, 128LL);
    long long ch = (K + chunks - 1) / chunks;
    return (ch + 63) / 64 * 64;
}

long long sgemm_kchunk(int M, int N, long long K, int sms) {
    const long long tiles = (long long)((M + SG_BM - 1) / SG_BM) * ((N + SG_BN - 1) / SG_BN);
    long long splits = 1;
    if (tiles < 2LL * sms) splits = std::min((2LL * sms + tiles - 1) / tiles, std::max(1LL, K / 256));
    splits = std::max(1LL, std::min(splits, 128LL));
    long long chunk = (K + splits - 1) / splits;
    return (chunk + SG_BK - 1) / SG_BK * SG_BK;
}

}  // namespace

int sgemm_splits(int M, int N, long long K, int sms, bool ta) {
    if (K <= 0) return 1;
    if (N <= 16) {
        if (!ta) return 1;
        const long long ch = narrow_kchunk(M, K, sms);
        return (int)((K + ch - 1) / ch);
    }
    const long long ch = sgemm_kchunk(M, N, K, sms);
    return (int)((K + ch - 1) / ch);
}

bool launch_sgemm(bool ta, bool tb, int M, int N, long long K, const float* A, long long lda, const float* B,
                  long long ldb, float beta, float* C, long long ldc, float* part, int sms, cudaStream_t stream,
                  int* launches) {
    if (M <= 0 || N <= 0 || K <= 0) return false;
    SgArgs a{M, N, K, A, lda, B, ldb, ta ? 1 : 0, tb ? 1 : 0, beta, C, ldc, nullptr, 0};
    int splits = 1;
    if (N <= 16) {
        if (!ta) {
            const int blocks = (int)std::min<long long>(((long long)M * 32 + 255) / 256, 16LL * sms);
            if (N <= 2) sgemm_narrow_rows<2><<<blocks, 256, 0, stream>>>(a);
            else if (N <= 4) sgemm_narrow_rows<4><<<blocks, 256, 0, stream>>>(a);
            else if (N <= 8) sgemm_narrow_rows<8><<<blocks, 256, 0, stream>>>(a);
            else sgemm_narrow_rows<16><<<blocks, 256, 0, stream>>>(a);
        } else {
            a.kchunk = narrow_kchunk(M, K, sms);
            splits = (int)((K + a.kchunk - 1) / a.kchunk);
            if (splits > 1) {
                if (!part) return false;
                a.part = part;
            }
            dim3 grid((unsigned)((M + 255) / 256), (unsigned)splits);
            if (N <= 2) sgemm_narrow_cols<2><<<grid, 256, 0, stream>>>(a);
            else if (N <= 4) sgemm_narrow_cols<4><<<grid, 256, 0, stream>>>(a);
            else if (N <= 8) sgemm_narrow_cols<8><<<grid, 256, 0, stream>>>(a);
            else sgemm_narrow_cols<16><<<grid, 256, 0, stream>>>(a);
        }
    } else {
        a.kchunk = sgemm_kchunk(M, N, K, sms);
        splits = (int)((K + a.kchunk - 1) / a.kchunk);
        if (splits > 1) {
            if (!part) return false;
            a.part = part;
        }
        dim3 grid((unsigned)((N + SG_BN - 1) / SG_BN), (unsigned)((M + SG_BM - 1) / SG_BM), (unsigned)splits);
        if (grid.y > 65535) return false;
        sgemm_tile<<<grid, 256, 0, stream>>>(a);
    }
    if (cudaGetLastError() != cudaSuccess) return false;
    int n = 1;
    if (splits > 1) {
        const long long tot = (long long)M * N;
        const int blocks = (int)std::min<long long>((tot + 255) / 256, 8LL * sms);
        if (splits >= 16 && tot <= 65536)
            sgemm_reduce_warp<<<(unsigned)((tot * 32 + 255) / 256), 256, 0, stream>>>(part, splits, M, N, C, ldc, beta);
        else
            sgemm_reduce<<<blocks, 256, 0, stream>>>(part, splits, M, N, C, ldc, beta);
        if (cudaGetLastError() != cudaSuccess) return false;
        ++n;
    }
    if (launches) *launches += n;
    return true;
}

}  // namespace ksb

// ---------------------------------------------------------------------------
// C-ABI: the training GEMM as a library call on caller device buffers
// ---------------------------------------------------------------------------
#include "ks_b200.h"
#include "ks_internal.h"

extern "C" ks_status ks_gemm_f16x3(int32_t ta, int32_t tb, int64_t M, int64_t N, int64_t K, const float* A,
                                   int64_t lda, const float* B, int64_t ldb, float beta, float* C, int64_t ldc,
                                   void* stream) {
    using ksb_host::set_error;
    if (M <= 0 || N <= 0 || K <= 0) return set_error(KS_ERR_SHAPE, "ks_gemm_f16x3: empty GEMM");
    if (beta != 0.0f && beta != 1.0f) return set_error(KS_ERR_PARAMETER, "ks_gemm_f16x3: beta must be 0 or 1");
    if (M > (1LL << 30) || N > (1LL << 30)) return set_error(KS_ERR_SHAPE, "ks_gemm_f16x3: M, N too large");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // planes in the operands' own layouts: A is M x K (or K x M when ta), B is K x N (or N x K when tb)
    const long long ar = ta ? K : M, ac = ta ? M : K, br = tb ? N : K, bc = tb ? K : N;
    const long long lda16 = (ac + 7) / 8 * 8, ldb16 = (bc + 7) / 8 * 8;
    const int splits = ksb::gemm16_splits((int)M, (int)N, K, sms);
    const size_t abytes = (size_t)ar * lda16 * 4, bbytes = (size_t)br * ldb16 * 4;  // hi + lo planes
    const size_t pbytes = splits > 1 ? (size_t)splits * M * N * 4 : 0;
    char* ws = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&ws), 256 + abytes + bbytes + pbytes, s);
    if (e != cudaSuccess) return set_error(KS_ERR_CUDA, std::string("ks_gemm_f16x3: ") + cudaGetErrorString(e));
    int* amax = reinterpret_cast<int*>(ws);       // [0] A, [1] B
    float* betad = reinterpret_cast<float*>(ws + 16);
    __half* a_hi = reinterpret_cast<__half*>(ws + 256);
    __half* a_lo = a_hi + (size_t)ar * lda16;
    __half* b_hi = reinterpret_cast<__half*>(ws + 256 + abytes);
    __half* b_lo = b_hi + (size_t)br * ldb16;
    float* part = pbytes ? reinterpret_cast<float*>(ws + 256 + abytes + bbytes) : nullptr;
    const float bsc[1] = {beta};
    cudaMemsetAsync(amax, 0, 8, s);
    cudaMemcpyAsync(betad, bsc, 4, cudaMemcpyHostToDevice, s);
    ksb::launch_absmax(A, ar, ac, lda, amax, s);
    ksb::launch_absmax(B, br, bc, ldb, amax + 1, s);
    ksb::launch_split_planes(A, ar, ac, lda, a_hi, a_lo, lda16, amax, s);
    ksb::launch_split_planes(B, br, bc, ldb, b_hi, b_lo, ldb16, amax + 1, s);
    ksb::GemmF16Args g{a_hi, a_lo, lda16, ta ? 1 : 0, b_hi, b_lo, ldb16, tb ? 0 : 1, (int)M, (int)N, K,
                       amax, amax + 1, betad, C, ldc, part, sms};
    const bool ok = ksb::launch_gemm16(g, s, nullptr);
    e = cudaFreeAsync(ws, s);
    if (!ok) return set_error(KS_ERR_CUDA, "ks_gemm_f16x3: tensor-core GEMM launch failed");
    if (e != cudaSuccess || (e = cudaGetLastError()) != cudaSuccess)
        return set_error(KS_ERR_CUDA, std::string("ks_gemm_f16x3: ") + cudaGetErrorString(e));
    return KS_OK;
}
