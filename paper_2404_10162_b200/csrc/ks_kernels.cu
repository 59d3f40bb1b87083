// ks_kernels.cu -- CUDA-core kernels of the B200 beam-decode engine:
//   * lstm_step_simt   fp32 gate GEMM + fused LSTM cell (FP32 precision mode,
//                      and the encoder's first step in every mode)
//   * attention_pack   additive attention + context, writes the decoder GEMM
//                      operand [ctx ; h_prev] (fp32 or fp16 hi/lo split)
//   (uatt = b_h + a_t . W_a is computed by the position-0 attention launch)
//   * beam_step        head GEMV + fp64 log-softmax + typed predicate mask +
//                      warp top-k with the reference tie-break
//   * beam_init        position-0 beam state
//
// Reference semantics restated (paths under /root/reference/proj):
//   lstm_cell_step        src/nn.cpp:88-128
//   attention_weights     src/models.cpp:265-281
//   context_vector        src/models.cpp:283-294
//   SequencePredictor::step src/models.cpp:448-493
//   beam_search_impl      src/decoding.cpp:27-103 (children, 1e-300 floor, predicate
//                         order, BeamExhaustedError, sort by (lp desc, prefix asc))
//   greedy_decode         src/decoding.cpp:107-124 (strict '>' argmax)
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdlib>

#include "ks_common.cuh"

namespace ksb {

__device__ __forceinline__ float sigmoidf_(float x) { return 1.0f / (1.0f + expf(-x)); }

__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max_f(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// ---------------------------------------------------------------------------
// Fused LSTM cell epilogue shared by the SIMT and tensor-core GEMMs.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void lstm_cell_store(const LstmArgs& p, int row, int u, float gi,
                                                float gf, float go, float gc, int slot,
                                                int crow) {
    const float* G = p.G + (long long)slot * 4 * p.H;
    gi += G[u];
    gf += G[p.H + u];
    go += G[2 * p.H + u];
    gc += G[3 * p.H + u];
    float cprev = 0.0f;
    if (p.c_prev != nullptr && crow >= 0) cprev = p.c_prev[(long long)crow * p.ldc_prev + u];
    const float ig = sigmoidf_(gi);
    const float fg = sigmoidf_(gf);
    const float og = sigmoidf_(go);
    const float cg = tanhf(gc);
    const float c = fg * cprev + ig * cg;
    const float h = og * tanhf(c);
    p.c_out[(long long)row * p.ldc + u] = c;
    p.h_out[(long long)row * p.ldh + u] = h;
    if (p.h_out2 != nullptr) p.h_out2[(long long)row * p.ldh2 + u] = h;
    if (p.hA_hi != nullptr) store_split_h(p, (long long)row * p.ldha + u, h);
}

__device__ __forceinline__ int row_slot(const LstmArgs& p, int row) {
    return p.slot_base + (p.slot_ptr ? p.slot_ptr[(long long)row * p.slot_stride] : 0);
}
__device__ __forceinline__ int row_crow(const LstmArgs& p, int row) {
    return p.parent ? p.parent[row] : row;
}

// ---------------------------------------------------------------------------
// lstm_cell_k0: an LSTM step with no dense input (K = 0: the first encoder
// step, zero state), i.e. gates = G[slot] -- pure elementwise, 4 units per
// thread with 128-bit loads/stores; same cell arithmetic as lstm_cell_store.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) lstm_cell_k0(LstmArgs a0, LstmArgs a1) {
    const LstmArgs& p = blockIdx.y == 0 ? a0 : a1;
    const int H4 = p.H >> 2;
    const long long n = (long long)p.M * H4;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int row = (int)(i / H4), u = (int)(i - (long long)row * H4) * 4;
        const float* G = p.G + (long long)row_slot(p, row) * 4 * p.H + u;
        const float4 gi = *reinterpret_cast<const float4*>(G);
        const float4 gf = *reinterpret_cast<const float4*>(G + p.H);
        const float4 go = *reinterpret_cast<const float4*>(G + 2 * p.H);
        const float4 gc = *reinterpret_cast<const float4*>(G + 3 * p.H);
        const int crow = row_crow(p, row);
        float4 cp = make_float4(0.f, 0.f, 0.f, 0.f);
        if (p.c_prev != nullptr && crow >= 0) cp = *reinterpret_cast<const float4*>(p.c_prev + (long long)crow * p.ldc_prev + u);
        const float I[4] = {gi.x, gi.y, gi.z, gi.w}, F[4] = {gf.x, gf.y, gf.z, gf.w};
        const float O[4] = {go.x, go.y, go.z, go.w}, Cg[4] = {gc.x, gc.y, gc.z, gc.w};
        const float Cp[4] = {cp.x, cp.y, cp.z, cp.w};
        float c[4], h[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            c[j] = sigmoidf_(F[j]) * Cp[j] + sigmoidf_(I[j]) * tanhf(Cg[j]);
            h[j] = sigmoidf_(O[j]) * tanhf(c[j]);
        }
        *reinterpret_cast<float4*>(p.c_out + (long long)row * p.ldc + u) = make_float4(c[0], c[1], c[2], c[3]);
        *reinterpret_cast<float4*>(p.h_out + (long long)row * p.ldh + u) = make_float4(h[0], h[1], h[2], h[3]);
        if (p.h_out2 != nullptr)
            *reinterpret_cast<float4*>(p.h_out2 + (long long)row * p.ldh2 + u) = make_float4(h[0], h[1], h[2], h[3]);
        if (p.hA_hi != nullptr) {
            const long long idx = (long long)row * p.ldha + u;
            if (p.ha_bf16) {
                __align__(8) __nv_bfloat16 hb[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) hb[j] = __float2bfloat16_rn(h[j]);
                *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(p.hA_hi) + idx) = *reinterpret_cast<const uint2*>(hb);
            } else {
                __align__(8) __half hh[4], hl[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) split_f16(h[j], hh[j], hl[j]);
                *reinterpret_cast<uint2*>(p.hA_hi + idx) = *reinterpret_cast<const uint2*>(hh);
                *reinterpret_cast<uint2*>(p.hA_lo + idx) = *reinterpret_cast<const uint2*>(hl);
            }
        }
    }
}

bool lstm_k0_ok(const LstmArgs& p) {
    auto al = [](const void* q, int b) { return (reinterpret_cast<uintptr_t>(q) & (uintptr_t)(b - 1)) == 0; };
    return p.K == 0 && p.H % 4 == 0 && al(p.G, 16) && p.ldc % 4 == 0 && p.ldh % 4 == 0 && al(p.c_out, 16) &&
           al(p.h_out, 16) && (p.c_prev == nullptr || (p.ldc_prev % 4 == 0 && al(p.c_prev, 16))) &&
           (p.h_out2 == nullptr || (p.ldh2 % 4 == 0 && al(p.h_out2, 16))) &&
           (p.hA_hi == nullptr || (p.ldha % 4 == 0 && al(p.hA_hi, 8) && (p.ha_bf16 || al(p.hA_lo, 8))));
}

bool launch_lstm_k0(const LstmArgs& a0, const LstmArgs* a1, int sms, cudaStream_t s) {
    if (!lstm_k0_ok(a0) || (a1 && (!lstm_k0_ok(*a1) || a1->M != a0.M || a1->H != a0.H))) return false;
    const long long n = (long long)a0.M * (a0.H / 4);
    const unsigned gx = (unsigned)std::max<long long>(1, std::min<long long>((n + 255) / 256, (long long)sms * 8));
    lstm_cell_k0<<<dim3(gx, a1 ? 2u : 1u), 256, 0, s>>>(a0, a1 ? *a1 : a0);
    return cudaGetLastError() == cudaSuccess;
}

// ---------------------------------------------------------------------------
// lstm_step_simt: tile 64 rows x 32 hidden units (x4 gates), 256 threads,
// K chunks of 32 through shared memory, 4x(2 units x 4 gates) per thread.
// ---------------------------------------------------------------------------
constexpr int SB_M = 64, SB_U = 32, SB_K = 32;

__global__ void __launch_bounds__(256) lstm_step_simt(LstmArgs a0, LstmArgs a1) {
    const LstmArgs& p = blockIdx.z == 0 ? a0 : a1;
    __shared__ float As[SB_K][SB_M + 1];
    __shared__ __align__(16) float Ws[SB_K][SB_U * 4];
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
    const int row0 = blockIdx.x * SB_M;
    const int ublk = blockIdx.y * SB_U;
    if (ublk >= p.H) return;
    float acc[4][8];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;

    for (int k0 = 0; k0 < p.K; k0 += SB_K) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int idx = tid + 256 * i;
            const int r = idx >> 5, kk = idx & 31;
            const int row = row0 + r;
            As[kk][r] = row < p.M ? p.A[(long long)row * p.lda + k0 + kk] : 0.0f;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int idx = tid + 256 * i;          // float4 index within 32 x 128
            const int kk = idx >> 5, c4 = idx & 31;
            const float4 v = *reinterpret_cast<const float4*>(
                p.W + (long long)(k0 + kk) * 4 * p.H + ublk * 4 + c4 * 4);
            *reinterpret_cast<float4*>(&Ws[kk][c4 * 4]) = v;
        }
        __syncthreads();
#pragma unroll 8
        for (int kk = 0; kk < SB_K; ++kk) {
            float a[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
            const float4 w0 = *reinterpret_cast<const float4*>(&Ws[kk][tx * 8]);
            const float4 w1 = *reinterpret_cast<const float4*>(&Ws[kk][tx * 8 + 4]);
            const float w[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], w[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int row = row0 + ty * 4 + i;
        if (row >= p.M) continue;
        const int slot = row_slot(p, row);
        const int crow = row_crow(p, row);
#pragma unroll
        for (int uu = 0; uu < 2; ++uu) {
            const int u = ublk + tx * 2 + uu;
            lstm_cell_store(p, row, u, acc[i][uu * 4 + 0], acc[i][uu * 4 + 1], acc[i][uu * 4 + 2],
                            acc[i][uu * 4 + 3], slot, crow);
        }
    }
}

// ---------------------------------------------------------------------------
// attention_pack: one warp per decoder row (models.cpp:265-294, 466-478).
//   s = h_prev[parent(row)] (zero state at position 0)
//   e_t = b_o + sum_d tanh(s.W_s[:,d] + u[t][d]) * w_o[d],  u[t][d] = b_h[d] + a_t.W_a[:,d]
//   alpha = softmax_t(e);  ctx = sum_t alpha_t a_t
//   A[row] = [ctx ; s]  (fp32, fp16 hi/lo split, or bf16)
// FIRST (position 0, one row per config): also computes and stores u.
// ---------------------------------------------------------------------------
template <int SPLIT>
__device__ __forceinline__ void store4p(float* A, __half* A_hi, __half* A_lo, long long idx, float4 v) {
    if (SPLIT == 0) {
        *reinterpret_cast<float4*>(A + idx) = v;
    } else if (SPLIT == 1) {
        __half2 h01, l01, h23, l23;
        split_f16x2(v.x, v.y, h01, l01);
        split_f16x2(v.z, v.w, h23, l23);
        uint2 h, l;
        h.x = *reinterpret_cast<uint32_t*>(&h01);
        h.y = *reinterpret_cast<uint32_t*>(&h23);
        l.x = *reinterpret_cast<uint32_t*>(&l01);
        l.y = *reinterpret_cast<uint32_t*>(&l23);
        *reinterpret_cast<uint2*>(A_hi + idx) = h;
        *reinterpret_cast<uint2*>(A_lo + idx) = l;
    } else {
        __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y);
        __nv_bfloat162 b = __floats2bfloat162_rn(v.z, v.w);
        uint2 h;
        h.x = *reinterpret_cast<uint32_t*>(&a);
        h.y = *reinterpret_cast<uint32_t*>(&b);
        *reinterpret_cast<uint2*>(A_hi + idx) = h;
    }
}
template <int SPLIT>
__device__ __forceinline__ void store4(const AttnArgs& p, long long idx, float4 v) {
    store4p<SPLIT>(p.A, p.A_hi, p.A_lo, idx, v);
}

// Alpha-block operand of the projected-context GEMM (row r of config b): the
// first kalpha columns hold alpha_t at 7 * (b - b0) + t, b0 = first config of
// r's 128-row tile, zeros elsewhere (written by the lanes of one warp).
template <int SPLIT>
__device__ __forceinline__ void write_alpha_block(const AttnArgs& p, int r, int b, const float (&al)[kTin],
                                                  int lane) {
    // column of alpha_0 = 7 * b - x0, x0 = 7 * b0 rounded down to 8 (see tile_k, ks_gemm_tc.cu)
    int b0 = (r / p.alpha_tile * p.alpha_tile) / p.H_rows;
    int width = p.kalpha;
    if (p.cp_cfg) {  // compacted rows: the tile's configs from the row -> config map
        const int Mv = *p.cp_M;
        const int t0 = r / p.alpha_tile * p.alpha_tile;
        const int last = (t0 + p.alpha_tile < Mv ? t0 + p.alpha_tile : Mv) - 1;
        b0 = p.cp_cfg[t0];
        const int cols = kTin * (p.cp_cfg[last] + 1) - ((kTin * b0) & ~7);
        width = (cols + 63) / 64 * 64;  // the K-blocks the GEMM contracts for this tile
        width = width < p.kalpha ? width : p.kalpha;
    }
    const int c0 = kTin * b - ((kTin * b0) & ~7);
    const long long base = (long long)r * (p.kalpha + p.NS);
    if (p.alpha_sparse) {  // the previous position left this layout's zeros in place
        if (lane < kTin) {
            float x = al[0];
#pragma unroll
            for (int t = 1; t < kTin; ++t) x = lane == t ? al[t] : x;
            if (SPLIT == 1) {
                __half hi, lo;
                split_f16s(x, kAlphaScale, hi, lo);
                p.A_hi[base + c0 + lane] = hi;
                p.A_lo[base + c0 + lane] = lo;
            } else {
                reinterpret_cast<__nv_bfloat16*>(p.A_hi)[base + c0 + lane] = __float2bfloat16_rn(x);
            }
        }
        return;
    }
    for (int c = lane; c < width / 8; c += 32) {
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int idx = 8 * c + j - c0;
            float x = 0.0f;
#pragma unroll
            for (int t = 0; t < kTin; ++t) x = idx == t ? al[t] : x;
            v[j] = x;
        }
        if (SPLIT == 1) {
            __align__(16) __half hi[8], lo[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) split_f16s(v[j], kAlphaScale, hi[j], lo[j]);
            *reinterpret_cast<uint4*>(p.A_hi + base + 8 * c) = *reinterpret_cast<const uint4*>(hi);
            *reinterpret_cast<uint4*>(p.A_lo + base + 8 * c) = *reinterpret_cast<const uint4*>(lo);
        } else {
            __align__(16) __nv_bfloat16 hb[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) hb[j] = __float2bfloat16_rn(v[j]);
            *reinterpret_cast<uint4*>(p.A_hi + base + 8 * c) = *reinterpret_cast<const uint4*>(hb);
        }
    }
}

template <int ND, int SPLIT, bool FIRST>
__device__ __forceinline__ void attention_row(const AttnArgs& p, int r, int lane) {
    const int b = p.cp_cfg ? p.cp_cfg[r] : r / p.H_rows;
    const int par = p.cp_prow ? p.cp_prow[r] : p.parent ? p.parent[r] : r;
    const float* s = (p.h_prev != nullptr && par >= 0) ? p.h_prev + (long long)par * p.ldh : nullptr;
    const int Kd = p.kalpha ? p.kalpha + p.NS : p.NA2 + p.NS;
    const int hc = p.kalpha ? p.kalpha : p.NA2;  // column of h_prev in the operand
    const long long base = (long long)r * Kd;
    float sd[ND > 0 ? ND : 1];
#pragma unroll
    for (int d = 0; d < ND; ++d) sd[d] = 0.0f;
#pragma unroll 4
    for (int c = lane; c < p.NS / 4; c += 32) {
        const float4 v = s ? *reinterpret_cast<const float4*>(s + 4 * c) : make_float4(0.f, 0.f, 0.f, 0.f);
        if (ND > 0 && s) {
            // the 4 W_s rows of this chunk are 4*ND contiguous floats: vector loads
            const float vv[4] = {v.x, v.y, v.z, v.w};
            float w[4 * (ND > 0 ? ND : 1)];
#pragma unroll
            for (int q = 0; q < ND; ++q) {
                const float4 w4 = reinterpret_cast<const float4*>(p.Ws + 4 * c * ND)[q];
                w[4 * q] = w4.x; w[4 * q + 1] = w4.y; w[4 * q + 2] = w4.z; w[4 * q + 3] = w4.w;
            }
            if (ND == 2) {  // paired FMAs: (sd0, sd1) += v_e (w_e0, w_e1)
                float2 acc2 = make_float2(sd[0], sd[ND - 1]);
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    acc2 = __ffma2_rn(make_float2(vv[e], vv[e]), make_float2(w[e * ND], w[e * ND + ND - 1]), acc2);
                sd[0] = acc2.x;
                sd[ND - 1] = acc2.y;
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e)
#pragma unroll
                    for (int d = 0; d < ND; ++d) sd[d] = fmaf(vv[e], w[e * ND + d], sd[d]);
            }
        }
        store4<SPLIT>(p, base + hc + 4 * c, v);
    }
    if (ND == 0) return;  // enc-dec: the operand is h_prev only
#pragma unroll
    for (int d = 0; d < ND; ++d) sd[d] = warp_sum_f(sd[d]);
    const float* act = p.act + (long long)b * kTin * p.NA2;
    float u[kTin][ND > 0 ? ND : 1];
    if (FIRST) {
#pragma unroll
        for (int t = 0; t < kTin; ++t) {
            float acc[ND > 0 ? ND : 1];
#pragma unroll
            for (int d = 0; d < ND; ++d) acc[d] = 0.0f;
#pragma unroll 4
            for (int c = lane; c < p.NA2 / 4; c += 32) {
                const float4 a4 = *reinterpret_cast<const float4*>(act + t * p.NA2 + 4 * c);
                const float av[4] = {a4.x, a4.y, a4.z, a4.w};
                float w[4 * (ND > 0 ? ND : 1)];
#pragma unroll
                for (int q = 0; q < ND; ++q) {
                    const float4 w4 = reinterpret_cast<const float4*>(p.Wa + 4 * c * ND)[q];
                    w[4 * q] = w4.x; w[4 * q + 1] = w4.y; w[4 * q + 2] = w4.z; w[4 * q + 3] = w4.w;
                }
#pragma unroll
                for (int e = 0; e < 4; ++e)
#pragma unroll
                    for (int d = 0; d < ND; ++d) acc[d] = fmaf(av[e], w[e * ND + d], acc[d]);
            }
#pragma unroll
            for (int d = 0; d < ND; ++d) {
                u[t][d] = warp_sum_f(acc[d]) + p.bh[d];
                if (lane == 0) p.uatt_out[((long long)b * kTin + t) * ND + d] = u[t][d];
            }
        }
    } else {
#pragma unroll
        for (int t = 0; t < kTin; ++t)
#pragma unroll
            for (int d = 0; d < ND; ++d) u[t][d] = p.uatt[((long long)b * kTin + t) * ND + d];
    }
    // e_t on lane t: b_o + sum_d tanh(s.W_s[:,d] + u[t][d]) w_o[d]; softmax over
    // lanes 0..7 (lane 7 carries exp = 0)
    float ev = -FLT_MAX;
    if (lane < kTin) {
        float v = p.bo;
#pragma unroll
        for (int d = 0; d < ND; ++d) {
            float ut = u[0][d];
#pragma unroll
            for (int t = 1; t < kTin; ++t) ut = lane == t ? u[t][d] : ut;
            v = fmaf(tanhf(sd[d] + ut), p.wo[d], v);
        }
        ev = v;
    }
    float mx = ev;
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const float ex = lane < kTin ? expf(ev - mx) : 0.0f;
    float sum = ex;
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const float al_lane = ex * (1.0f / sum);
    float e[kTin];
#pragma unroll
    for (int t = 0; t < kTin; ++t) e[t] = __shfl_sync(0xffffffffu, al_lane, t);
    if (SPLIT != 0 && p.kalpha) {  // projected context: alpha . P^T on the tensor cores
        write_alpha_block<SPLIT>(p, r, b, e, lane);
        return;
    }
    for (int c = lane; c < p.NA2 / 4; c += 32) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int t = 0; t < kTin; ++t) {
            const float4 a4 = *reinterpret_cast<const float4*>(act + t * p.NA2 + 4 * c);
            acc.x = fmaf(e[t], a4.x, acc.x);
            acc.y = fmaf(e[t], a4.y, acc.y);
            acc.z = fmaf(e[t], a4.z, acc.z);
            acc.w = fmaf(e[t], a4.w, acc.w);
        }
        store4<SPLIT>(p, base + 4 * c, acc);
    }
}

template <int ND, int SPLIT, bool FIRST>
__global__ void __launch_bounds__(256) attention_pack_t(AttnArgs p) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // persistent: one warp per row, grid-strided (the grid is sized to one resident wave);
    // compacted rows: *cp_M of them
    const int M = p.cp_M ? *p.cp_M : p.M;
    for (int r = blockIdx.x * (blockDim.x >> 5) + warp; r < M; r += gridDim.x * (blockDim.x >> 5))
        attention_row<ND, SPLIT, FIRST>(p, r, lane);
}

// Config-per-warp variant for positions > 0: the H rows of a config share
// a_t, so each a_t chunk is loaded once and reused for all rows (G at a time).
template <int ND, int SPLIT>
__global__ void __launch_bounds__(256, 3) attention_cfg_t(AttnArgs p) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int H = p.H_rows;
    const int b = blockIdx.x * (blockDim.x >> 5) + warp;
    if ((long long)b * H >= p.M) return;
    const int Kd = p.kalpha ? p.kalpha + p.NS : p.NA2 + p.NS;
    const int hc = p.kalpha ? p.kalpha : p.NA2;
    const float* act = p.act + (long long)b * kTin * p.NA2;
    constexpr int G = 4;
    for (int i0 = 0; i0 < H; i0 += G) {
        const int ng = H - i0 < G ? H - i0 : G;
        float al[G][kTin];
#pragma unroll
        for (int ii = 0; ii < G; ++ii) {
            if (ii >= ng) break;
            const int r = b * H + i0 + ii;
            const int par = p.parent ? p.parent[r] : r;
            const float* sh = (p.h_prev != nullptr && par >= 0) ? p.h_prev + (long long)par * p.ldh : nullptr;
            float sd[ND > 0 ? ND : 1];
#pragma unroll
            for (int d = 0; d < ND; ++d) sd[d] = 0.0f;
#pragma unroll 4
            for (int c = lane; c < p.NS / 4; c += 32) {
                const float4 v = sh ? *reinterpret_cast<const float4*>(sh + 4 * c) : make_float4(0.f, 0.f, 0.f, 0.f);
                const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int e = 0; e < 4; ++e)
#pragma unroll
                    for (int d = 0; d < ND; ++d) sd[d] = fmaf(vv[e], p.Ws[(4 * c + e) * ND + d], sd[d]);
                store4<SPLIT>(p, (long long)r * Kd + hc + 4 * c, v);
            }
            if (ND == 0) continue;
#pragma unroll
            for (int d = 0; d < ND; ++d) sd[d] = warp_sum_f(sd[d]);
            float mx = -FLT_MAX;
#pragma unroll
            for (int t = 0; t < kTin; ++t) {
                float v = p.bo;
#pragma unroll
                for (int d = 0; d < ND; ++d)
                    v = fmaf(tanhf(sd[d] + p.uatt[((long long)b * kTin + t) * ND + d]), p.wo[d], v);
                al[ii][t] = v;
                mx = fmaxf(mx, v);
            }
            float sum = 0.0f;
#pragma unroll
            for (int t = 0; t < kTin; ++t) {
                al[ii][t] = expf(al[ii][t] - mx);
                sum += al[ii][t];
            }
            const float inv = 1.0f / sum;
#pragma unroll
            for (int t = 0; t < kTin; ++t) al[ii][t] *= inv;
            if (SPLIT != 0 && p.kalpha) {
                float a7[kTin];
#pragma unroll
                for (int t = 0; t < kTin; ++t) a7[t] = al[ii][t];
                write_alpha_block<SPLIT>(p, r, b, a7, lane);
            }
        }
        if (ND == 0 || p.kalpha) continue;
#pragma unroll 2
        for (int c = lane; c < p.NA2 / 4; c += 32) {
            float4 at[kTin];
#pragma unroll
            for (int t = 0; t < kTin; ++t) at[t] = *reinterpret_cast<const float4*>(act + t * p.NA2 + 4 * c);
#pragma unroll
            for (int ii = 0; ii < G; ++ii) {
                if (ii >= ng) break;
                float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int t = 0; t < kTin; ++t) {
                    acc.x = fmaf(al[ii][t], at[t].x, acc.x);
                    acc.y = fmaf(al[ii][t], at[t].y, acc.y);
                    acc.z = fmaf(al[ii][t], at[t].z, acc.z);
                    acc.w = fmaf(al[ii][t], at[t].w, acc.w);
                }
                store4<SPLIT>(p, (long long)(b * H + i0 + ii) * Kd + 4 * c, acc);
            }
        }
    }
}

// CTA-per-config variant (positions > 0): 4 warps; warp w scores rows w, w+4,
// ... (s . W_s, energies, softmax -> alpha in shared memory), then every
// thread owns a float4 column of a_t, loads its 7 steps once and writes the
// context of all H rows of the config.
template <int ND, int SPLIT>
__global__ void __launch_bounds__(128) attention_cta_t(AttnArgs p) {
    constexpr int kMaxRows = 64;
    __shared__ float alpha[kMaxRows][kTin];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int H = p.H_rows;
    const int b = blockIdx.x;
    const int Kd = p.kalpha ? p.kalpha + p.NS : p.NA2 + p.NS;
    const int hc = p.kalpha ? p.kalpha : p.NA2;
    for (int i = warp; i < H; i += 4) {
        const int r = b * H + i;
        const int par = p.parent ? p.parent[r] : r;
        const float* sh = (p.h_prev != nullptr && par >= 0) ? p.h_prev + (long long)par * p.ldh : nullptr;
        float sd[ND > 0 ? ND : 1];
#pragma unroll
        for (int d = 0; d < ND; ++d) sd[d] = 0.0f;
#pragma unroll 4
        for (int c = lane; c < p.NS / 4; c += 32) {
            const float4 v = sh ? *reinterpret_cast<const float4*>(sh + 4 * c) : make_float4(0.f, 0.f, 0.f, 0.f);
            const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int e = 0; e < 4; ++e)
#pragma unroll
                for (int d = 0; d < ND; ++d) sd[d] = fmaf(vv[e], p.Ws[(4 * c + e) * ND + d], sd[d]);
            store4<SPLIT>(p, (long long)r * Kd + hc + 4 * c, v);
        }
        if (ND == 0) continue;
#pragma unroll
        for (int d = 0; d < ND; ++d) sd[d] = warp_sum_f(sd[d]);
        float e[kTin];
        float mx = -FLT_MAX;
#pragma unroll
        for (int t = 0; t < kTin; ++t) {
            float v = p.bo;
#pragma unroll
            for (int d = 0; d < ND; ++d)
                v = fmaf(tanhf(sd[d] + p.uatt[((long long)b * kTin + t) * ND + d]), p.wo[d], v);
            e[t] = v;
            mx = fmaxf(mx, v);
        }
        float sum = 0.0f;
#pragma unroll
        for (int t = 0; t < kTin; ++t) {
            e[t] = expf(e[t] - mx);
            sum += e[t];
        }
        const float inv = 1.0f / sum;
        if (SPLIT != 0 && p.kalpha) {
#pragma unroll
            for (int t = 0; t < kTin; ++t) e[t] *= inv;
            write_alpha_block<SPLIT>(p, r, b, e, lane);
            continue;
        }
        if (lane < kTin) {
            float my = e[0];
#pragma unroll
            for (int t = 1; t < kTin; ++t)
                if (lane == t) my = e[t];
            alpha[i][lane] = my * inv;
        }
    }
    if (ND == 0 || p.kalpha) return;
    __syncthreads();
    const float* act = p.act + (long long)b * kTin * p.NA2;
    for (int c = threadIdx.x; c < p.NA2 / 4; c += blockDim.x) {
        float4 at[kTin];
#pragma unroll
        for (int t = 0; t < kTin; ++t) at[t] = *reinterpret_cast<const float4*>(act + t * p.NA2 + 4 * c);
        for (int i = 0; i < H; ++i) {
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int t = 0; t < kTin; ++t) {
                const float al = alpha[i][t];
                acc.x = fmaf(al, at[t].x, acc.x);
                acc.y = fmaf(al, at[t].y, acc.y);
                acc.z = fmaf(al, at[t].z, acc.z);
                acc.w = fmaf(al, at[t].w, acc.w);
            }
            store4<SPLIT>(p, (long long)(b * H + i) * Kd + 4 * c, acc);
        }
    }
}

template <int ND, int SPLIT>
void launch_attention_nd(const AttnArgs& p, bool first, cudaStream_t s) {
    // KS_ATTN_MODE: 0 = CTA per config (default), 1 = warp per row, 2 = warp per config
    static const int mode = [] {
        const char* e = std::getenv("KS_ATTN_MODE");
        return e ? std::atoi(e) : 0;
    }();
    // warp-per-row kernel: persistent grid of one resident wave
    auto wave = [](void (*kern)(AttnArgs), long long want) -> unsigned {
        int per_sm = 0, sms = 148, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0) != cudaSuccess || per_sm < 1)
            per_sm = 1;
        return (unsigned)std::max<long long>(1, std::min<long long>(want, (long long)sms * per_sm));
    };
    if (first) {
        attention_pack_t<ND, SPLIT, true><<<wave(attention_pack_t<ND, SPLIT, true>, (p.M + 7) / 8), 256, 0, s>>>(p);
    } else if (mode == 0 && p.H_rows > 1 && p.H_rows <= 64 && p.kalpha == 0 && !p.cp_M) {
        attention_cta_t<ND, SPLIT><<<(unsigned)(p.M / p.H_rows), 128, 0, s>>>(p);
    } else if (mode == 2 && p.H_rows > 1 && !p.cp_M) {
        const int C = p.M / p.H_rows;
        attention_cfg_t<ND, SPLIT><<<(unsigned)((C + 7) / 8), 256, 0, s>>>(p);
    } else {
        attention_pack_t<ND, SPLIT, false><<<wave(attention_pack_t<ND, SPLIT, false>, (p.M + 7) / 8), 256, 0, s>>>(p);
    }
}

template <int SPLIT>
bool launch_attention_split(const AttnArgs& p, bool first, cudaStream_t s) {
    switch (p.nd) {
        case 0: launch_attention_nd<0, SPLIT>(p, first, s); return true;
        case 1: launch_attention_nd<1, SPLIT>(p, first, s); return true;
        case 2: launch_attention_nd<2, SPLIT>(p, first, s); return true;
        case 3: launch_attention_nd<3, SPLIT>(p, first, s); return true;
        case 4: launch_attention_nd<4, SPLIT>(p, first, s); return true;
        case 5: launch_attention_nd<5, SPLIT>(p, first, s); return true;
        case 6: launch_attention_nd<6, SPLIT>(p, first, s); return true;
        case 7: launch_attention_nd<7, SPLIT>(p, first, s); return true;
        case 8: launch_attention_nd<8, SPLIT>(p, first, s); return true;
        default: return false;
    }
}

bool launch_attention(const AttnArgs& p, bool first, cudaStream_t s) {
    if (p.split_mode == 0) return launch_attention_split<0>(p, first, s);
    if (p.split_mode == 1) return launch_attention_split<1>(p, first, s);
    return launch_attention_split<2>(p, first, s);
}

// ---------------------------------------------------------------------------
// split_rows: fp32 -> the tensor-core operand planes (fp16 hi/lo or bf16),
// for the encoder activations a_t feeding the context projection P.
// ---------------------------------------------------------------------------
template <int SPLIT>
__global__ void split_rows_t(const float* src, long long n4, __half* hi, __half* lo) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x)
        store4p<SPLIT>(nullptr, hi, lo, 4 * i, reinterpret_cast<const float4*>(src)[i]);
}

bool launch_split_rows(const float* src, long long n, __half* hi, __half* lo, int mode, cudaStream_t s) {
    const long long n4 = n / 4;
    const unsigned grid = (unsigned)std::min<long long>((n4 + 255) / 256, 148 * 16);
    if (mode == 1)
        split_rows_t<1><<<grid, 256, 0, s>>>(src, n4, hi, lo);
    else
        split_rows_t<2><<<grid, 256, 0, s>>>(src, n4, hi, lo);
    return cudaGetLastError() == cudaSuccess;
}

// ---------------------------------------------------------------------------
// topk_eval: topk_metrics' per-sample scoring on the device (eval.cpp:117-134,
// 142-146): the best-matching beam (most matching positions, ties to the
// higher-ranked beam) adds its per-position hits; a sample counts as perfect
// if any of its beams matches every position.  One thread per config; the
// integer sums go through shared memory and one atomic per block and counter.
// ---------------------------------------------------------------------------
__global__ void topk_eval(const int* out_tok, const int* count, const int* truth, int B, int k, int T,
                          unsigned long long* pos_matches, unsigned long long* perfect) {
    __shared__ unsigned int s_pos[kMaxT];
    __shared__ unsigned int s_perf;
    for (int i = threadIdx.x; i < T; i += blockDim.x) s_pos[i] = 0;
    if (threadIdx.x == 0) s_perf = 0;
    __syncthreads();
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < B) {
        const int* tr = truth + (long long)b * T;
        const int n = count[b];
        int best = -1, best_m = -1;
        bool perf = false;
        for (int j = 0; j < n; ++j) {
            const int* bt = out_tok + ((long long)b * k + j) * T;
            int m = 0;
            for (int p = 0; p < T; ++p) m += bt[p] == tr[p];
            perf = perf || m == T;
            if (m > best_m) {
                best_m = m;
                best = j;
            }
        }
        if (best >= 0) {
            const int* bt = out_tok + ((long long)b * k + best) * T;
            for (int p = 0; p < T; ++p)
                if (bt[p] == tr[p]) atomicAdd(&s_pos[p], 1u);
        }
        if (perf) atomicAdd(&s_perf, 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < T; i += blockDim.x)
        if (s_pos[i]) atomicAdd(&pos_matches[i], (unsigned long long)s_pos[i]);
    if (threadIdx.x == 0 && s_perf) atomicAdd(perfect, (unsigned long long)s_perf);
}

bool launch_topk_eval(const int* out_tok, const int* count, const int* truth, int B, int k, int T,
                      unsigned long long* pos_matches, unsigned long long* perfect, cudaStream_t s) {
    if (T > kMaxT) return false;
    topk_eval<<<(unsigned)((B + 255) / 256), 256, 0, s>>>(out_tok, count, truth, B, k, T, pos_matches, perfect);
    return cudaGetLastError() == cudaSuccess;
}

// ---------------------------------------------------------------------------
// beam_init: position 0 has one live hypothesis per config (decoding.cpp:41-43).
// ---------------------------------------------------------------------------
__global__ void beam_init(int B, unsigned char* live, double* lp, unsigned long long* key,
                          int* status, int* fail_pred, int* fail_step) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    live[b] = 1;
    lp[b] = 0.0;
    key[b] = 0ull;
    status[b] = 0;
    fail_pred[b] = -1;
    fail_step[b] = -1;
}

// ---------------------------------------------------------------------------
// beam_step: one warp per config.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int key_token(unsigned long long key, const PosMeta& m, int i) {
    return (int)((key >> m.shift[i]) & ((1ull << m.bits[i]) - 1ull));
}

// Predicate programs and the output-value table, staged in shared memory once
// per CTA (they are read for every candidate).
struct PredTables {
    const DevPred* preds;
    const unsigned char* pred_bytes;
    const int* term_pos;
    const double* term_w;
    const int* term_field;
    const long long* values;
};

__device__ __forceinline__ size_t pred_tables_bytes(const BeamArgs& a) {
    size_t n = (size_t)a.n_values * 8 + (size_t)a.n_terms * 8;
    n += (size_t)a.n_preds * sizeof(DevPred);
    n += (size_t)a.n_terms * 8 + (size_t)a.n_bytes;
    return (n + 15) & ~(size_t)15;
}

__device__ PredTables stage_pred_tables(const BeamArgs& a, unsigned char* base) {
    long long* values = reinterpret_cast<long long*>(base);
    double* tw = reinterpret_cast<double*>(values + a.n_values);
    DevPred* preds = reinterpret_cast<DevPred*>(tw + a.n_terms);
    int* tpos = reinterpret_cast<int*>(preds + a.n_preds);
    int* tfield = tpos + a.n_terms;
    unsigned char* bytes = reinterpret_cast<unsigned char*>(tfield + a.n_terms);
    for (int i = threadIdx.x; i < a.n_values; i += blockDim.x) values[i] = a.values[i];
    for (int i = threadIdx.x; i < a.n_terms; i += blockDim.x) {
        tw[i] = a.term_w[i];
        tpos[i] = a.term_pos[i];
        tfield[i] = a.term_field[i];
    }
    for (int i = threadIdx.x; i < a.n_preds; i += blockDim.x) preds[i] = a.preds[i];
    for (int i = threadIdx.x; i < a.n_bytes; i += blockDim.x) bytes[i] = a.pred_bytes[i];
    return PredTables{preds, bytes, tpos, tw, tfield, values};
}

__device__ bool pred_accepts(const PredTables& a, const PosMeta& m, const DevPred& q,
                             unsigned long long key, int pos, const long long* desc_b) {
    switch (q.kind) {
        case 1: {  // MASK
            // Every earlier token of a live hypothesis already passed this (per-token)
            // predicate at its own position, so only the new token needs checking --
            // unless the predicate is full-sequence-only and runs just once, at the end.
            const unsigned char* allowed = a.pred_bytes + q.allowed_off;
            for (int i = q.full ? 0 : pos; i <= pos; ++i)
                if (!allowed[m.value_offset[i] + key_token(key, m, i)]) return false;
            return true;
        }
        case 2: {  // BUDGET: alphabetical terms, separate fp64 mul and add (constraints.cpp:234-239)
            double cost = 0.0;
            for (int t = 0; t < q.n_terms; ++t) {
                const int pp = a.term_pos[q.terms_off + t];
                if (pp < 0 || pp > pos) continue;
                const double v = (double)a.values[m.value_offset[pp] + key_token(key, m, pp)];
                cost = __dadd_rn(cost, __dmul_rn(a.term_w[q.terms_off + t], v));
            }
            return cost <= q.budget;
        }
        case 3: {  // PRODUCT
            __int128 prod = q.scale;
            const __int128 cap = (__int128)1 << 100;
            for (int t = 0; t < q.n_terms; ++t) {
                const int pp = a.term_pos[q.terms_off + t];
                if (pp < 0 || pp > pos) continue;
                prod *= (__int128)a.values[m.value_offset[pp] + key_token(key, m, pp)];
                if (prod > cap) prod = cap;
                if (prod < -cap) prod = -cap;
            }
            return prod <= (__int128)q.limit;
        }
        case 4: {  // DIVIDES (per-token like MASK: earlier tokens already passed)
            for (int t = 0; t < q.n_terms; ++t) {
                const int pp = a.term_pos[q.terms_off + t];
                if (pp < 0 || pp > pos || (!q.full && pp != pos)) continue;
                const long long v = a.values[m.value_offset[pp] + key_token(key, m, pp)];
                if (v <= 0 || desc_b == nullptr) return false;
                if (desc_b[a.term_field[q.terms_off + t]] % v != 0) return false;
            }
            return true;
        }
        default:
            return true;
    }
}


// Order-preserving unsigned image of an fp64 score (-0.0 folded onto +0.0 so
// that it compares equal, as in better()); 0 is never produced for a non-NaN.
__device__ __forceinline__ unsigned long long order_key(double s) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(s + 0.0);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// Candidate order: higher score first, exact ties to the smaller packed
// prefix key (= lexicographically smaller prefix; Candidate::operator<,
// decoding.cpp:21-24).
__device__ __forceinline__ bool better(double s1, unsigned long long k1, double s2,
                                       unsigned long long k2) {
    return s1 > s2 || (s1 == s2 && k1 < k2);
}

// Reduce-scatter of VP per-lane partial sums over the warp: after it, the
// lane src_lane<VP>(v) holds the full 32-lane sum for token v.  Costs
// VP-1 + (5 - log2 VP) shuffles instead of 5*VP for independent reductions.
template <int VP>
struct RS {
    static constexpr int L = VP == 32 ? 5 : VP == 16 ? 4 : VP == 8 ? 3 : 2;
};
template <int VP>
__device__ __forceinline__ float reduce_scatter(float (&p)[VP], int lane) {
    constexpr int L = RS<VP>::L;
#pragma unroll
    for (int l = 0; l < L; ++l) {
        const int mask = 16 >> l;
        const int half = VP >> (l + 1);
        const bool hi = (lane & mask) != 0;
#pragma unroll
        for (int j = 0; j < half; ++j) {
            const float keep = hi ? p[half + j] : p[j];
            const float send = hi ? p[j] : p[half + j];
            p[j] = keep + __shfl_xor_sync(0xffffffffu, send, mask);
        }
    }
    float v = p[0];
#pragma unroll
    for (int l = L; l < 5; ++l) v += __shfl_xor_sync(0xffffffffu, v, 16 >> l);
    return v;
}
template <int VP>
__device__ __forceinline__ int src_lane(int v) {
    constexpr int L = RS<VP>::L;
    int lane = 0;
#pragma unroll
    for (int l = 0; l < L; ++l) lane |= ((v >> (L - 1 - l)) & 1) << (4 - l);
    return lane;
}

template <int VP>
__global__ void __launch_bounds__(256, VP == 32 ? 1 : VP == 16 ? 2 : 4) beam_step_t(BeamArgs a, PosMeta m) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int WS = VP == 4 ? 12 : VP + 4;  // padded W row: conflict-free 128-bit loads
    const int V = m.vsize[a.pos];
    float* Wsh = reinterpret_cast<float*>(smem);
    // NS % 4 == 0: hidden rows are read as float4 (lane owns elements 4q..4q+3), so
    // W row i is stored at slot (i % 4) * NS/4 + i / 4 -- for a fixed component the
    // lanes then read consecutive slots, conflict-free like the scalar layout.
    const bool v4 = (a.NS & 3) == 0 && (reinterpret_cast<uintptr_t>(a.h) & 15) == 0;
    const int NQ = a.NS >> 2;
    for (int i = threadIdx.x; i < a.NS * VP; i += blockDim.x) {
        const int row = i / VP, v = i - row * VP;
        const int slot = v4 ? (row & 3) * NQ + (row >> 2) : row;
        Wsh[slot * WS + v] = v < V ? a.Wh[row * V + v] : 0.0f;
    }
    const size_t wbytes = ((size_t)a.NS * WS * 4 + 15) & ~(size_t)15;
    const PredTables tabs = stage_pred_tables(a, smem + wbytes);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    unsigned char* cbase = smem + wbytes + pred_tables_bytes(a) + (size_t)warp * a.cands_per_warp * 28;
    double* c_score = reinterpret_cast<double*>(cbase);
    double* c_lp = c_score + a.cands_per_warp;
    unsigned long long* c_key = reinterpret_cast<unsigned long long*>(c_lp + a.cands_per_warp);
    int* c_meta = reinterpret_cast<int*>(c_key + a.cands_per_warp);
    const int nc = a.H_cur * V;
    const int T = m.T;
    const float bias = lane < V ? a.bh[lane] : 0.0f;
    const int my_src = src_lane<VP>(lane < VP ? lane : 0);

    for (int b = blockIdx.x * nwarps + warp; b < a.B; b += gridDim.x * nwarps) {
        const long long* desc_b = a.desc ? a.desc + (long long)b * kTin : nullptr;
        auto write_dead_next = [&](int from) {
            if (a.final_step) return;
            for (int i = from + lane; i < a.H_next; i += 32) {
                const long long sl = (long long)b * a.H_next + i;
                a.live_next[sl] = 0;
                a.lp_next[sl] = -INFINITY;
                a.key_next[sl] = 0ull;
                a.parent_next[sl] = b * a.H_cur;
                a.slot_next[sl] = m.fb_offset[a.pos];
            }
        };
        if (a.status[b] != 0) {  // exhausted earlier: nothing left to extend
            write_dead_next(0);
            continue;
        }
        int n_alive = 0;
        int last_live = -1;
        for (int j0 = 0; j0 < a.H_cur; j0 += 2) {
            const long long r0 = (long long)b * a.H_cur + j0;
            const bool two = j0 + 1 < a.H_cur;
            const bool live0 = a.live_cur[r0] != 0;
            const bool live1 = two && a.live_cur[r0 + 1] != 0;
            if (!live0 && !live1) {
                for (int c = lane; c < (two ? 2 : 1) * V; c += 32) c_meta[j0 * V + c] = -1;
                continue;
            }
            // head logits for rows j0, j0+1: logits[v] = b[v] + sum_i h[i] W[i][v]  (models.cpp:490-491)
            float lg[2] = {0.0f, 0.0f};
            {
                // paired fp32 FMAs (FFMA2: two exact fp32 fma.rn per instruction)
                float2 q0[VP / 2], q1[VP / 2];
#pragma unroll
                for (int v = 0; v < VP / 2; ++v) {
                    q0[v] = make_float2(0.0f, 0.0f);
                    q1[v] = make_float2(0.0f, 0.0f);
                }
                // hybrid variants: every hypothesis of config b reads the same feature row
                const float* h0 = a.h + (a.h_per_config ? (long long)b : r0) * a.NS;
                const float* h1 = a.h_per_config ? h0 : h0 + a.NS;
                auto fma_row = [&](float x0, float x1, const float4* w4) {
                    const float2 X0 = make_float2(x0, x0), X1 = make_float2(x1, x1);
#pragma unroll
                    for (int qq = 0; qq < VP / 4; ++qq) {
                        const float4 w = w4[qq];
                        const float2 wa = make_float2(w.x, w.y), wb = make_float2(w.z, w.w);
                        q0[2 * qq] = __ffma2_rn(X0, wa, q0[2 * qq]);
                        q0[2 * qq + 1] = __ffma2_rn(X0, wb, q0[2 * qq + 1]);
                        q1[2 * qq] = __ffma2_rn(X1, wa, q1[2 * qq]);
                        q1[2 * qq + 1] = __ffma2_rn(X1, wb, q1[2 * qq + 1]);
                    }
                };
                if (v4) {
                    // 128-bit loads, both rows' loads in flight together; the next pair's
                    // rows (or the warp's next config's first pair) are prefetched into L2
                    // meanwhile
                    if (!a.h_per_config) {
                        const long long rn = j0 + 2 < a.H_cur ? r0 + 2
                                             : (long long)(b + gridDim.x * nwarps) * a.H_cur;
                        const int nrows = j0 + 2 < a.H_cur ? (j0 + 3 < a.H_cur ? 2 : 1)
                                          : (b + gridDim.x * nwarps < a.B ? (a.H_cur > 1 ? 2 : 1) : 0);
                        for (int q = lane; q < NQ * nrows; q += 32)
                            asm volatile("prefetch.global.L2 [%0];" ::"l"(a.h + rn * a.NS + 4 * q));
                    }
                    const float4* h04 = reinterpret_cast<const float4*>(h0);
                    const float4* h14 = reinterpret_cast<const float4*>(h1);
                    const float4 z4 = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll 4
                    for (int q = lane; q < NQ; q += 32) {
                        const float4 x0 = live0 ? __ldg(h04 + q) : z4;
                        const float4 x1 = live1 ? __ldg(h14 + q) : z4;
                        fma_row(x0.x, x1.x, reinterpret_cast<const float4*>(Wsh + (0 * NQ + q) * WS));
                        fma_row(x0.y, x1.y, reinterpret_cast<const float4*>(Wsh + (1 * NQ + q) * WS));
                        fma_row(x0.z, x1.z, reinterpret_cast<const float4*>(Wsh + (2 * NQ + q) * WS));
                        fma_row(x0.w, x1.w, reinterpret_cast<const float4*>(Wsh + (3 * NQ + q) * WS));
                    }
                } else {
#pragma unroll(VP <= 8 ? 16 : 4)
                    for (int i = lane; i < a.NS; i += 32)
                        fma_row(live0 ? h0[i] : 0.0f, live1 ? h1[i] : 0.0f,
                                reinterpret_cast<const float4*>(Wsh + i * WS));
                }
                float p0[VP], p1[VP];
#pragma unroll
                for (int v = 0; v < VP / 2; ++v) {
                    p0[2 * v] = q0[v].x;
                    p0[2 * v + 1] = q0[v].y;
                    p1[2 * v] = q1[v].x;
                    p1[2 * v + 1] = q1[v].y;
                }
                const float s0 = reduce_scatter<VP>(p0, lane);
                const float s1 = reduce_scatter<VP>(p1, lane);
                lg[0] = __shfl_sync(0xffffffffu, s0, my_src);
                lg[1] = __shfl_sync(0xffffffffu, s1, my_src);
            }
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
                const int j = j0 + jj;
                if (j >= a.H_cur) break;
                const bool live = jj == 0 ? live0 : live1;
                if (!live) {
                    for (int v = lane; v < V; v += 32) c_meta[j * V + v] = -1;
                    continue;
                }
                last_live = j;
                // log-softmax (nn.cpp:215-226) as (l - max) - log(sum exp), i.e. log(p)
                // without underflow, floored at log(1e-300) like decoding.cpp:57-58; the
                // hypothesis score accumulates in fp64
                const float l = lane < V ? lg[jj] + bias : -INFINITY;
                const float mx = warp_max_f(l);
                const float ex = lane < V ? expf(l - mx) : 0.0f;
                const float sum = warp_sum_f(ex);
                if (lane < V) {
                    const float lpt = fmaxf((l - mx) - logf(sum), -690.77552789821368f);
                    const double clp = a.lp_cur[r0 + jj] + (double)lpt;
                    const int c = j * V + lane;
                    // model_forward: the softmax (nn.cpp:215-226) of this position
                    if (a.out_dist) a.out_dist[(long long)b * a.dist_ld + a.dist_off + lane] = (double)(ex / sum);
                    // greedy_decode's argmax of p == argmax of the logit (ties -> lowest index);
                    // teacher forcing feeds back the teacher's token instead
                    c_score[c] = a.greedy ? (a.teacher ? (lane == a.teacher[(long long)b * T + a.pos] ? 1.0 : 0.0)
                                                       : (double)l)
                                          : clp;
                    c_lp[c] = clp;
                    c_meta[c] = 0;  // live, predicates pending
                }
            }
        }
        __syncwarp();
        // Constraint predicates over all H_cur x V children at once, 32 per pass
        // (lane-dense even when V < 32).
        for (int c0 = 0; c0 < nc; c0 += 32) {
            const int c = c0 + lane;
            int rej = -1;
            bool ok = false;
            if (c < nc && c_meta[c] == 0) {
                const int j = c / V, v = c - j * V;
                const long long r = (long long)b * a.H_cur + j;
                const unsigned long long key = a.key_cur[r] | ((unsigned long long)v << m.shift[a.pos]);
                // host-evaluated (opaque) predicates: registration index of the first
                // rejecting one; typed predicates registered before it still win
                const int hrej = a.host_rej ? a.host_rej[r * V + v] : -1;
                const int qend = hrej >= 0 ? hrej : a.n_preds;
                rej = hrej;
                for (int q = 0; q < qend; ++q) {
                    const DevPred& pq = tabs.preds[q];
                    if (pq.kind == 5) continue;  // KS_PRED_HOST: decided by the hook
                    if (pq.full && !a.final_step) continue;
                    if (!pred_accepts(tabs, m, pq, key, a.pos, desc_b)) {
                        rej = q;
                        break;
                    }
                }
                c_key[c] = key;
                c_meta[c] = rej < 0 ? ((j << 8) | v) : -2 - rej;
                ok = rej < 0;
            }
            n_alive += __popc(__ballot_sync(0xffffffffu, ok));
        }
        __syncwarp();
        if (n_alive == 0) {
            // BeamExhaustedError(last_rejecting, pos): every child was rejected, so the
            // last rejecting predicate is that of the last child (last live hyp, last token).
            if (lane == 0) {
                int fp = -1;
                if (last_live >= 0) {
                    const int mm = c_meta[last_live * V + V - 1];
                    fp = mm <= -2 ? -2 - mm : -1;
                }
                a.status[b] = 1;
                a.fail_pred[b] = fp;
                a.fail_step[b] = a.pos;
                a.out_count[b] = 0;
                if (a.out_status) a.out_status[b] = 1;
                if (a.out_fail_pred) a.out_fail_pred[b] = fp;
                if (a.out_fail_step) a.out_fail_step[b] = a.pos;
            }
            for (int i = lane; i < a.k * T; i += 32) a.out_tok[(long long)b * a.k * T + i] = -1;
            for (int i = lane; i < a.k; i += 32) a.out_lp[(long long)b * a.k + i] = -INFINITY;
            write_dead_next(0);
            __syncwarp();
            continue;
        }
        const int ksel = n_alive < a.k ? n_alive : a.k;
        // k rounds of warp argmax; each lane caches the best of its own candidates
        // and only the lane that owned the winner rescans.  The argmax runs on the
        // order-preserving 64-bit image of the fp64 score with two redux.sync maxima
        // (high word, then low word among the lanes holding that high word); exact
        // score ties fall back to the smallest prefix key the same way.
        double bs = -INFINITY;
        unsigned long long bk = ~0ull;
        int bc = -1;
        auto rescan = [&]() {
            bs = -INFINITY;
            bk = ~0ull;
            bc = -1;
            for (int c = lane; c < nc; c += 32) {
                if (c_meta[c] < 0) continue;
                if (bc < 0 || better(c_score[c], c_key[c], bs, bk)) {
                    bs = c_score[c];
                    bk = c_key[c];
                    bc = c;
                }
            }
        };
        rescan();
        for (int i = 0; i < ksel; ++i) {
            const unsigned long long u = bc < 0 ? 0ull : order_key(bs);
            const unsigned uh = (unsigned)(u >> 32), ul = (unsigned)u;
            const unsigned mh = __reduce_max_sync(0xffffffffu, uh);
            const unsigned ml = __reduce_max_sync(0xffffffffu, uh == mh ? ul : 0u);
            unsigned tie = __ballot_sync(0xffffffffu, bc >= 0 && uh == mh && ul == ml);
            if (tie & (tie - 1)) {  // equal scores: smaller packed prefix key wins
                const bool in = (tie >> lane) & 1u;
                const unsigned kh = (unsigned)(bk >> 32), kl = (unsigned)bk;
                const unsigned nh = __reduce_min_sync(0xffffffffu, in ? kh : 0xffffffffu);
                const unsigned nl = __reduce_min_sync(0xffffffffu, in && kh == nh ? kl : 0xffffffffu);
                tie = __ballot_sync(0xffffffffu, in && kh == nh && kl == nl);
            }
            const int wl = __ffs(tie) - 1;
            if (lane == wl) {  // this lane owns the winner (prefix keys are unique)
                const int meta = c_meta[bc];
                const int j = meta >> 8, v = meta & 255;
                const double clp = c_lp[bc];
                if (a.final_step) {
                    const long long o = (long long)b * a.k + i;
                    a.out_lp[o] = clp;
                    for (int t = 0; t < T; ++t) a.out_tok[o * T + t] = key_token(bk, m, t);
                } else {
                    const long long sl = (long long)b * a.H_next + i;
                    a.live_next[sl] = 1;
                    a.lp_next[sl] = clp;
                    a.key_next[sl] = bk;
                    a.parent_next[sl] = b * a.H_cur + j;
                    a.slot_next[sl] = m.fb_offset[a.pos] + v;
                }
                c_meta[bc] = -1;
                rescan();
            }
        }
        __syncwarp();
        if (a.final_step) {
            for (int i = ksel + lane; i < a.k; i += 32) {
                const long long o = (long long)b * a.k + i;
                a.out_lp[o] = -INFINITY;
                for (int t = 0; t < T; ++t) a.out_tok[o * T + t] = -1;
            }
            if (lane == 0) {
                a.out_count[b] = ksel;
                if (a.out_status) a.out_status[b] = 0;
                if (a.out_fail_pred) a.out_fail_pred[b] = -1;
                if (a.out_fail_step) a.out_fail_step[b] = -1;
            }
        } else {
            write_dead_next(ksel);
        }
        __syncwarp();
    }
}

size_t beam_smem_bytes(int NS, int V, int warps, int cands_per_warp, size_t tables) {
    const int VP = V <= 4 ? 4 : V <= 8 ? 8 : V <= 16 ? 16 : 32;
    const int WS = VP == 4 ? 12 : VP + 4;
    return (((size_t)NS * WS * 4 + 15) & ~(size_t)15) + ((tables + 15) & ~(size_t)15) +
           (size_t)warps * cands_per_warp * 28;
}

bool launch_beam(const BeamArgs& a, const PosMeta& m, int warps, size_t smem, int grid, cudaStream_t s) {
    const int V = m.vsize[a.pos];
    static std::atomic<unsigned long long> attr{0};
    if (first_on_device(attr)) {
        cudaFuncSetAttribute(beam_step_t<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        cudaFuncSetAttribute(beam_step_t<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        cudaFuncSetAttribute(beam_step_t<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        cudaFuncSetAttribute(beam_step_t<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    }
    auto kern = V <= 4 ? beam_step_t<4> : V <= 8 ? beam_step_t<8> : V <= 16 ? beam_step_t<16> : beam_step_t<32>;
    // persistent grid: exactly the CTAs that fit at once (registers and shared memory
    // both limit residency; a partial second wave would leave most SMs idle)
    int per_sm = 0, dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, warps * 32, smem) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    const int g = std::min(grid, sms * per_sm);
    kern<<<g, warps * 32, smem, s>>>(a, m);
    return cudaGetLastError() == cudaSuccess;
}

}  // namespace ksb

namespace ksb {

// ---------------------------------------------------------------------------
// hybrid_conv: the hybrid variants' convolutional encoder (hybrid_encode,
// models.cpp:296-309; conv1d_forward, nn.cpp:171-213), one warp per config.
// Layer 0 reads the one-hot (d_in x 7) input matrix as gathers of the hot
// channel per time step; later layers are dense.  The flattened (f, o)
// encoding is written as the x part of the bi-LSTM operands (split or fp32)
// of both directions and both ping-pong buffers; the h part of buffer 0 is
// zeroed (zero initial state).
// ---------------------------------------------------------------------------


__global__ void __launch_bounds__(128) hybrid_conv(ConvArgs p) {
    extern __shared__ float cs[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.x * (blockDim.x >> 5) + warp;
    if (b >= p.C) return;
    float* buf0 = cs + (size_t)warp * 2 * p.scratch_floats;
    float* buf1 = buf0 + p.scratch_floats;
    int hot[kTin];
#pragma unroll
    for (int t = 0; t < kTin; ++t) hot[t] = p.in_offset[t] + p.tok[(long long)b * kTin + t];
    int ch = p.d_in, len = kTin;
    float* in = nullptr;
    float* out = buf0;
    for (int i = 0; i < p.n_conv; ++i) {
        const int f = p.f[i], k = p.k[i], st = p.s[i];
        const int o = (len - k) / st + 1;
        for (int idx = lane; idx < f * o; idx += 32) {
            const int ff = idx / o, j = idx - ff * o;
            float acc = p.b[i][ff];
            if (i == 0) {
                for (int u = 0; u < k; ++u) acc += p.W[0][((long long)ff * ch + hot[j * st + u]) * k + u];
            } else {
                for (int c = 0; c < ch; ++c)
                    for (int u = 0; u < k; ++u)
                        acc = fmaf(p.W[i][((long long)ff * ch + c) * k + u], in[c * len + j * st + u], acc);
            }
            out[idx] = acc;
        }
        __syncwarp();
        in = out;
        out = (out == buf0) ? buf1 : buf0;
        ch = f;
        len = o;
    }
    // x part of every operand buffer; zero h part of the step-0 buffers
    for (int q = 0; q < 4; ++q) {
        const long long base = (long long)b * p.K;
        for (int c = lane; c < p.FP + ((q & 1) == 0 ? p.CP : 0); c += 32) {
            const float v = c < p.F ? in[c] : 0.0f;
            if (p.split_mode == 0) {
                p.Af[q][base + c] = v;
            } else if (p.split_mode == 1) {
                __half hi, lo;
                split_f16(v, hi, lo);
                p.Ahi[q][base + c] = hi;
                p.Alo[q][base + c] = lo;
            } else {
                reinterpret_cast<__nv_bfloat16*>(p.Ahi[q])[base + c] = __float2bfloat16_rn(v);
            }
        }
    }
}

// hybrid: bi-LSTM 2 operand of step t = [fwd h1_t | bwd h1_t | h2]; the h2
// part of each direction's first step is the zero initial state, the others
// are written by bi-LSTM 2's own epilogue.
__global__ void hybrid_pack(HybPackArgs p) {
    const long long K2 = 3LL * p.CP;
    const long long n = (long long)p.T * p.C * K2;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long row = i / K2;
        const int col = (int)(i - row * K2);
        const int t = (int)(row / p.C);
        const bool hpart = col >= 2 * p.CP;
        const float v = hpart ? 0.0f : p.H1[row * 2 * p.CP + col];
        for (int dir = 0; dir < 2; ++dir) {
            if (hpart && t != (dir == 0 ? 0 : p.T - 1)) continue;
            if (p.split_mode == 0) {
                p.Xf[dir][i] = v;
            } else if (p.split_mode == 1) {
                __half hi, lo;
                split_f16(v, hi, lo);
                p.Xhi[dir][i] = hi;
                p.Xlo[dir][i] = lo;
            } else {
                reinterpret_cast<__nv_bfloat16*>(p.Xhi[dir])[i] = __float2bfloat16_rn(v);
            }
        }
    }
}

bool launch_hybrid_pack(const HybPackArgs& p, cudaStream_t s) {
    const long long n = (long long)p.T * p.C * 3 * p.CP;
    hybrid_pack<<<(unsigned)std::min<long long>((n + 255) / 256, 148LL * 64), 256, 0, s>>>(p);
    return cudaGetLastError() == cudaSuccess;
}

bool launch_hybrid_conv(const ConvArgs& p, cudaStream_t s) {
    const size_t smem = (size_t)4 * 2 * p.scratch_floats * sizeof(float);
    if (smem > 200 * 1024) return false;
    static std::atomic<unsigned long long> attr{0};
    if (first_on_device(attr)) cudaFuncSetAttribute(hybrid_conv, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    hybrid_conv<<<(unsigned)((p.C + 3) / 4), 128, smem, s>>>(p);
    return cudaGetLastError() == cudaSuccess;
}

}  // namespace ksb
