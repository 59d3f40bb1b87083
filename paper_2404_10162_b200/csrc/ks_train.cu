// ks_train.cu -- teacher-forced training step on the B200 (BASELINE config 4),
// behind the C-ABI ks_trainer_* (include/ks_b200.h).
//
// Reference: train_model's batch body (proj/src/models.cpp:905-947): per-sample
// build_loss_graph + Tape::backward (models.cpp:638-780, autodiff.cpp:326-544),
// gradients summed over the batch, / batch, clip_global_norm 5.0, adam_step
// (nn.cpp:262-297).  Here the batch is one set of rows on the device:
//
//   forward   encoder bi-LSTM (7 steps per direction), attention + post LSTM
//             (T steps), heads + cross entropy; every step is one fp32 GEMM
//             (cuBLAS) + one fused elementwise kernel; activations are kept
//             for the backward pass (~1.3 GB at batch 4096, default model).
//   backward  BPTT in reverse: fused cell-backward / attention-backward
//             kernels + one dX GEMM per step; all weight gradients of an LSTM
//             are ONE GEMM over every (step, row) pair at the end
//             (X_all^T . dZ_all), one-hot input rows and the bias as one GEMM
//             against a (mask-scaled) slot-indicator matrix.
//   dropout   train_model's variational masks, drawn on the device from the
//             reference's own stream Rng::derive(seed, epoch << 32 | idx)
//             (models.cpp:915-918, LstmMasks::make 559-573): mt19937_64 per
//             sample, bit-identical to the reference's masks.
//   apply     grads / batch, global-norm clip, Adam (fp64 arithmetic per
//             element; fp32 parameters and moments).
//
// Multi-GPU: ks_trainer_loss_grads writes per-rank SUMMED gradients into a
// caller-owned flat buffer; the host all-reduces it (NCCL via
// torch.distributed) and every rank calls ks_trainer_apply with the global
// batch -- the placement SURVEY.md §5 gives for the reference's in-process
// gradient sum (models.cpp:936-945).
//
// Parameter layout ("train layout", flat fp32): reference tensors in
// alphabetical (checkpoint) order, except that each LSTM's eight tensors are
// packed as one segment  Wd [x_dense + H][4H]  (dense input rows, then the
// recurrent rows; column g*H + j, gates input, forget, output, cand)  followed
// by  Ws [S + 1][4H]  (one-hot slot rows, then the bias).  Adam and the clip
// are elementwise / order-free, so they run on the flat buffer directly.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include "ks_b200.h"
#include "ks_internal.h"
#include "ks_tc.cuh"

using ksb_host::set_error;

namespace kst {

constexpr int kTin = 7;
constexpr int kMaxNd = 8;
constexpr int kMaxT = 16;

// ---------------------------------------------------------------------------
// device kernels
// ---------------------------------------------------------------------------

// Rng::derive's seed mixing (rng.hpp:19-21, 64-68).
__device__ __forceinline__ unsigned long long rng_mix(unsigned long long z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
// One warp per sample: input mask (n_in) then recurrent mask (n_rec), as
// LstmMasks::make -> nn::dropout_mask draw them (nn.cpp:237-248).  The
// mt19937_64 state lives in shared memory; seeding is serial (lane 0), the
// twist runs in three dependency-respecting parallel phases (i < 156 reads only
// old words; 156 <= i < 311 reads old mt[i + 1] and the phase-1 results; i = 311
// reads the new mt[0]), and the 312 tempered outputs of a block go one per lane.
__device__ __forceinline__ unsigned long long mt_twist_one(const unsigned long long* mt, int i) {
    const unsigned long long x = (mt[i] & 0xFFFFFFFF80000000ULL) | (mt[(i + 1) % 312] & 0x7FFFFFFFULL);
    unsigned long long xa = x >> 1;
    if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
    return mt[(i + 156) % 312] ^ xa;
}
__global__ void k_set_u64x2(unsigned long long* d, unsigned long long a, unsigned long long b) {
    d[0] = a;
    d[1] = b;
}
__global__ void k_set_int(int* d, int v) { *d = v; }
__device__ __forceinline__ unsigned long long mt_temper(unsigned long long y) {
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    return y ^ (y >> 43);
}

// se = {seed, epoch} in device memory (written per step outside the captured graph)
__global__ void k_dropout_masks(int M, const unsigned long long* se, const long long* idx,
                                long long idx_base, int n_in, double rate_in, int n_rec, double rate_rec,
                                float* mi, float* mr) {
    __shared__ unsigned long long st[8][312];
    const unsigned long long seed = se[0];
    const long long epoch = (long long)se[1];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.x * (blockDim.x >> 5) + w;
    if (b >= M) return;
    unsigned long long* mt = st[w];
    if (lane == 0) {
        const unsigned long long id = idx ? (unsigned long long)idx[b] : (unsigned long long)(idx_base + b);
        const unsigned long long stream = ((unsigned long long)epoch << 32) | id;
        mt[0] = rng_mix(rng_mix(seed) + 0x9e3779b97f4a7c15ULL * (stream + 1));
        for (int i = 1; i < 312; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i;
    }
    __syncwarp();
    const float ki = (float)(1.0 / (1.0 - rate_in)), kr = (float)(1.0 / (1.0 - rate_rec));
    const int n = n_in + n_rec;
    for (int base = 0; base < n; base += 312) {
        unsigned long long v[5];
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            const int i = lane + 32 * q;
            if (i < 156) v[q] = mt_twist_one(mt, i);
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            const int i = lane + 32 * q;
            if (i < 156) mt[i] = v[q];
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            const int i = 156 + lane + 32 * q;
            if (i < 311) v[q] = mt_twist_one(mt, i);
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            const int i = 156 + lane + 32 * q;
            if (i < 311) mt[i] = v[q];
        }
        __syncwarp();
        if (lane == 0) mt[311] = mt_twist_one(mt, 311);
        __syncwarp();
        for (int e = lane; e < 312 && base + e < n; e += 32) {
            const int g = base + e;
            const double u = (double)(mt_temper(mt[e]) >> 11) * 0x1.0p-53;
            if (g < n_in)
                mi[(long long)b * n_in + g] = u < rate_in ? 0.0f : ki;
            else
                mr[(long long)b * n_rec + (g - n_in)] = u < rate_rec ? 0.0f : kr;
        }
        __syncwarp();
    }
}

// Slot ids / values per (step, row) and the slot-indicator matrices used by
// the one-hot + bias gradient GEMMs.
struct SlotArgs {
    int M, T, variant;
    const int* tok;  // [M][7]
    const int* tgt;  // [M][T]
    int in_off[kTin];
    int fb_off[kMaxT];
    int d_in, d_fb;
    int enc_dirs;
    int dec_slots;        // S of the decoder LSTM (0 for attn-2)
    int dec_mask_off;     // column of slot 0 in the decoder input mask
    int n_in;             // input-mask width
    const float* mi;      // [M][n_in] or null
    int* enc_slot;        // [7][M] by time t
    int* dec_slot;        // [T][M]
    float* dec_val;       // [T][M]
    float* enc_sm[2];     // [7][M][d_in + 1] per direction, rows in processing order
    float* dec_sm;        // [T][M][dec_slots + 1]
};

__global__ void k_slots(SlotArgs a) {
    const long long n_enc = (long long)kTin * a.M;
    const long long n_dec = (long long)a.T * a.M;
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (tid < n_enc) {
        const int t = (int)(tid / a.M), b = (int)(tid % a.M);
        const int slot = a.in_off[t] + a.tok[(long long)b * kTin + t];
        a.enc_slot[tid] = slot;
        for (int dir = 0; dir < a.enc_dirs; ++dir) {
            const int s = dir == 0 ? t : kTin - 1 - t;  // processing step of time t
            float* row = a.enc_sm[dir] + ((long long)s * a.M + b) * (a.d_in + 1);
            for (int k = 0; k <= a.d_in; ++k) row[k] = (k == slot || k == a.d_in) ? 1.0f : 0.0f;
        }
    } else if (tid < n_enc + n_dec) {
        const long long q = tid - n_enc;
        const int p = (int)(q / a.M), b = (int)(q % a.M);
        int slot = -1;
        float val = 0.0f;
        if (a.dec_slots > 0) {
            slot = p == 0 ? 0 : a.fb_off[p - 1] + a.tgt[(long long)b * a.T + p - 1];
            val = a.mi ? a.mi[(long long)b * a.n_in + a.dec_mask_off + slot] : 1.0f;
        }
        a.dec_slot[q] = slot;
        a.dec_val[q] = val;
        float* row = a.dec_sm + q * (a.dec_slots + 1);
        for (int k = 0; k < a.dec_slots; ++k) row[k] = k == slot ? val : 0.0f;
        row[a.dec_slots] = 1.0f;
    }
}

__device__ __forceinline__ float sigm(float x) { return 1.0f / (1.0f + expf(-x)); }

// Fused LSTM cell forward (tape_lstm_step, models.cpp:578-593):
// z = Z (GEMM of the dense rows, null = 0) + val * Ws[slot] + Ws[S] (bias);
// Z is overwritten with the activations (i, f, o, g) for the backward pass.
struct CellFwd {
    int M, H, S;
    float* Z;               // [M][4H] in: pre-activation (dense part), out: activations
    int zero_z;             // Z holds no GEMM result (all dense rows are zero)
    const float* Ws;        // [(S+1)][4H]
    const int* slot;        // [M] or null
    const float* val;       // [M] or null (1)
    const float* c_prev;    // [M][H] or null
    float* c_out;           // [M][H]
    float* h_out;           // unmasked h
    long long ldh;
    float* h_out2;          // optional second copy (next GEMM operand), masked by mr
    long long ldh2;
    const float* mr;        // [M][H] or null
    __half* q_hi;           // optional F16X3 planes of h_out2 (row stride ldq), scale from *qamax
    __half* q_lo;
    long long ldq;
    const int* qamax;
};

// one value into F16X3 planes (the k_split_planes rounding: hi = rn(x 2^e), lo = rn(x 2^e - hi))
__device__ __forceinline__ void store_planes(float v, float sc, __half* hi, __half* lo, long long i) {
    const float x = v * sc;
    const __half h = __float2half_rn(x);
    hi[i] = h;
    lo[i] = __float2half_rn(x - __half2float(h));
}

// four consecutive units of one row per thread (128-bit loads / stores along the
// units) when H and the row strides allow it, else one unit per thread
template <int VEC>
__global__ void k_cell_fwd(CellFwd a) {
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int HV = a.H / VEC;
    if (tid >= (long long)a.M * HV) return;
    const int r = (int)(tid / HV), j0 = (int)(tid % HV) * VEC;
    const int H = a.H;
    const float* bias = a.Ws + (long long)a.S * 4 * H;
    const int slot = a.slot ? a.slot[r] : -1;
    const float val = a.val ? a.val[r] : 1.0f;
    float* Zr = a.Z + (long long)r * 4 * H;
    float z[4][VEC];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        float zz[VEC], bb[VEC], ww[VEC];
        if (VEC == 4) {
            const float4 zv = a.zero_z ? make_float4(0.f, 0.f, 0.f, 0.f) : *reinterpret_cast<const float4*>(Zr + g * H + j0);
            const float4 bv = *reinterpret_cast<const float4*>(bias + g * H + j0);
            const float4 wv = slot >= 0 ? *reinterpret_cast<const float4*>(a.Ws + (long long)slot * 4 * H + g * H + j0)
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
            zz[0] = zv.x; zz[1] = zv.y; zz[2] = zv.z; zz[3] = zv.w;
            bb[0] = bv.x; bb[1] = bv.y; bb[2] = bv.z; bb[3] = bv.w;
            ww[0] = wv.x; ww[1] = wv.y; ww[2] = wv.z; ww[3] = wv.w;
        } else {
            zz[0] = a.zero_z ? 0.0f : Zr[g * H + j0];
            bb[0] = bias[g * H + j0];
            ww[0] = slot >= 0 ? a.Ws[(long long)slot * 4 * H + g * H + j0] : 0.0f;
        }
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
            float v = zz[e];
            if (slot >= 0) v += val * ww[e];
            z[g][e] = v + bb[e];
        }
    }
    float act[4][VEC], c[VEC], h[VEC], h2[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
        const int j = j0 + e;
        const float i = sigm(z[0][e]), f = sigm(z[1][e]), o = sigm(z[2][e]), g = tanhf(z[3][e]);
        const float cp = a.c_prev ? a.c_prev[(long long)r * H + j] : 0.0f;
        c[e] = f * cp + i * g;
        h[e] = o * tanhf(c[e]);
        act[0][e] = i;
        act[1][e] = f;
        act[2][e] = o;
        act[3][e] = g;
        h2[e] = a.mr ? h[e] * a.mr[(long long)r * H + j] : h[e];
    }
    if (VEC == 4) {
#pragma unroll
        for (int g = 0; g < 4; ++g)
            *reinterpret_cast<float4*>(Zr + g * H + j0) = make_float4(act[g][0], act[g][1], act[g][2], act[g][3]);
        *reinterpret_cast<float4*>(a.c_out + (long long)r * H + j0) = make_float4(c[0], c[1], c[2], c[3]);
        *reinterpret_cast<float4*>(a.h_out + (long long)r * a.ldh + j0) = make_float4(h[0], h[1], h[2], h[3]);
        if (a.h_out2)
            *reinterpret_cast<float4*>(a.h_out2 + (long long)r * a.ldh2 + j0) = make_float4(h2[0], h2[1], h2[2], h2[3]);
    } else {
#pragma unroll
        for (int g = 0; g < 4; ++g) Zr[g * H + j0] = act[g][0];
        a.c_out[(long long)r * H + j0] = c[0];
        a.h_out[(long long)r * a.ldh + j0] = h[0];
        if (a.h_out2) a.h_out2[(long long)r * a.ldh2 + j0] = h2[0];
    }
    if (a.h_out2 && a.q_hi) {
        const float qs = exp2f((float)ksb::f16_scale_exp(*a.qamax));
#pragma unroll
        for (int e = 0; e < VEC; ++e) store_planes(h2[e], qs, a.q_hi, a.q_lo, (long long)r * a.ldq + j0 + e);
    }
}

bool cell_fwd_vec_ok(const CellFwd& c) {
    auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    return c.H % 4 == 0 && c.ldh % 4 == 0 && (!c.h_out2 || (c.ldh2 % 4 == 0 && al(c.h_out2))) && al(c.Z) &&
           al(c.Ws) && al(c.c_out) && al(c.h_out);
}
void launch_cell_fwd(const CellFwd& c, cudaStream_t s) {
    if (cell_fwd_vec_ok(c))
        k_cell_fwd<4><<<(unsigned)(((long long)c.M * (c.H / 4) + 255) / 256), 256, 0, s>>>(c);
    else
        k_cell_fwd<1><<<(unsigned)(((long long)c.M * c.H + 255) / 256), 256, 0, s>>>(c);
}

// Fused LSTM cell backward: dh = dh1 + dh2 (* mask2); writes dZ (pre-activation
// gradients, the GEMM operand) and dc_prev in place of dc.
struct CellBwd {
    int M, H;
    const float* act;       // [M][4H] activations
    const float* c;         // [M][H]
    const float* c_prev;    // [M][H] or null
    const float* dh1;       // or null
    long long ld1;
    const float* dh2;       // or null
    long long ld2;
    const float* mask2;     // [M][H] or null, applied to dh2
    float* dc;              // [M][H] in: dc from the next step (zeroed at the end), out: dc_prev
    float* dZ;              // [M][4H]
    int* amax0;             // F16X3 trainer GEMMs: max |dZ| of this launch / of every step, or null
    int* amax1;
};

__device__ __forceinline__ void cell_bwd_elem(const CellBwd& a, long long tid, float& mx);
__global__ void __launch_bounds__(256) k_cell_bwd(CellBwd a) {
    float mx = 0.0f;
    for (long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x; tid < (long long)a.M * a.H;
         tid += (long long)gridDim.x * blockDim.x)
        cell_bwd_elem(a, tid, mx);
    if (a.amax0 == nullptr && a.amax1 == nullptr) return;
    // the max |dZ| the F16X3 split of the dX / dW GEMMs needs, one atomic per block
    __shared__ float wm[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x < 32) {
        mx = threadIdx.x < (blockDim.x >> 5) ? wm[threadIdx.x] : 0.0f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (threadIdx.x == 0 && mx > 0.0f) {
            if (a.amax0) atomicMax(a.amax0, __float_as_int(mx));
            if (a.amax1) atomicMax(a.amax1, __float_as_int(mx));
        }
    }
}
__device__ __forceinline__ void cell_bwd_elem(const CellBwd& a, long long tid, float& mx) {
    const int r = (int)(tid / a.H), j = (int)(tid % a.H);
    const int H = a.H;
    const float* A = a.act + (long long)r * 4 * H;
    const float i = A[j], f = A[H + j], o = A[2 * H + j], g = A[3 * H + j];
    const float c = a.c[(long long)r * H + j];
    const float cp = a.c_prev ? a.c_prev[(long long)r * H + j] : 0.0f;
    float dh = a.dh1 ? a.dh1[(long long)r * a.ld1 + j] : 0.0f;
    if (a.dh2) {
        const float d2 = a.dh2[(long long)r * a.ld2 + j];
        dh += a.mask2 ? d2 * a.mask2[(long long)r * H + j] : d2;
    }
    const float tc = tanhf(c);
    const float dc = a.dc[(long long)r * H + j] + dh * o * (1.0f - tc * tc);
    const float dout = dh * tc;
    float* dZ = a.dZ + (long long)r * 4 * H;
    const float z0 = dc * g * i * (1.0f - i), z1 = dc * cp * f * (1.0f - f);
    const float z2 = dout * o * (1.0f - o), z3 = dc * i * (1.0f - g * g);
    dZ[j] = z0;
    dZ[H + j] = z1;
    dZ[2 * H + j] = z2;
    dZ[3 * H + j] = z3;
    a.dc[(long long)r * H + j] = dc * f;
    mx = fmaxf(mx, fmaxf(fmaxf(fabsf(z0), fabsf(z1)), fmaxf(fabsf(z2), fabsf(z3))));
}

// Attention forward, one warp per row (the tape form of attention_weights +
// context_vector, models.cpp:700-712): e_t = wo . tanh(s.Ws + a_t.Wa + bh) + bo,
// alpha = softmax_t(e), ctx = sum_t alpha_t a_t; writes ctx (masked) into the
// ctx columns of the post-LSTM operand.
struct AttnFwd {
    int M, na2, ns, nd;
    const float* s;      // [M][ns] (h of the previous position, unmasked)
    const float* A;      // [M][7][na2]
    const float* U;      // [M][7][nd] = a_t . Wa (no bias)
    const float* Ws;     // [ns][nd]
    const float* bh;     // [nd]
    const float* wo;     // [nd]
    const float* bo;     // [1]
    const float* mi;     // [M][n_in] or null (ctx columns 0..na2)
    int n_in;
    float* X;            // [M][ldx], ctx written at columns 0..na2
    long long ldx;
    __half* x_hi;        // optional F16X3 planes of X (row stride ldxq), scale from *qamax
    __half* x_lo;
    long long ldxq;
    const int* qamax;
    float* alpha;        // [M][7]
    float* hid;          // [M][7][nd]
};

template <int ND>
__global__ void k_attn_fwd(AttnFwd a) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= a.M) return;
    const long long r = warp;
    const float* s = a.s + r * a.ns;
    float sw[ND];
    #pragma unroll
    for (int d = 0; d < ND; ++d) sw[d] = 0.0f;
    for (int j = lane; j < a.ns; j += 32) {
        const float sv = s[j];
        #pragma unroll
        for (int d = 0; d < ND; ++d) sw[d] += sv * a.Ws[(long long)j * ND + d];
    }
    #pragma unroll
    for (int d = 0; d < ND; ++d)
        for (int o = 16; o; o >>= 1) sw[d] += __shfl_xor_sync(0xffffffffu, sw[d], o);
    float e[kTin];
    float mx = -INFINITY;
    for (int t = 0; t < kTin; ++t) {
        float et = a.bo[0];
        #pragma unroll
        for (int d = 0; d < ND; ++d) {
            const float hv = tanhf(sw[d] + a.U[(r * kTin + t) * ND + d] + a.bh[d]);
            if (lane == 0) a.hid[(r * kTin + t) * ND + d] = hv;
            et += hv * a.wo[d];
        }
        e[t] = et;
        mx = fmaxf(mx, et);
    }
    float sum = 0.0f;
    for (int t = 0; t < kTin; ++t) {
        e[t] = expf(e[t] - mx);
        sum += e[t];
    }
    for (int t = 0; t < kTin; ++t) {
        e[t] /= sum;
        if (lane == 0) a.alpha[r * kTin + t] = e[t];
    }
    const float* Ar = a.A + r * kTin * a.na2;
    const float qsc = a.x_hi ? exp2f((float)ksb::f16_scale_exp(*a.qamax)) : 0.0f;
    for (int j = lane; j < a.na2; j += 32) {
        float c = 0.0f;
        for (int t = 0; t < kTin; ++t) c += e[t] * Ar[t * a.na2 + j];
        const float x = a.mi ? c * a.mi[r * a.n_in + j] : c;
        a.X[r * a.ldx + j] = x;
        if (a.x_hi) store_planes(x, qsc, a.x_hi, a.x_lo, r * a.ldxq + j);
    }
}

// Attention backward, one warp per row.  Input dX = [dctx | dh_rec] (the dX
// GEMM of the post LSTM); produces dH = dh_rec * mr + ds (ds through s.Ws),
// keeps this position's (masked) dctx for k_attn_dA, accumulates the per-row
// sums for attn.out and the dpre terms reduced later by GEMMs (DPs for Ws,
// DPa for Wa and bh).
struct AttnBwd {
    int M, na2, ns, nd;
    const float* dX;     // [M][ldx]
    long long ldx;
    const float* mi;     // [M][n_in] or null
    int n_in;
    const float* mr;     // [M][ns] or null
    const float* A;      // [M][7][na2]
    const float* alpha;  // [M][7]
    const float* hid;    // [M][7][nd]
    const float* Ws;     // [ns][nd]
    const float* Wa;     // [na2][nd]
    const float* wo;     // [nd]
    float* dctx_out;     // [M][na2] (=) this position's masked dctx
    float* dH;           // [M][ns] (=)
    float* DPs;          // [M][nd] (=) this position
    float* DPa;          // [M][7][nd] (+=)
    float* rowacc;       // [M][nd + 1] (+=): sum_t hid*de, sum_t de
};

template <int ND>
__global__ void k_attn_bwd(AttnBwd a) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= a.M) return;
    const long long r = warp;
    const float* dX = a.dX + r * a.ldx;
    const float* Ar = a.A + r * kTin * a.na2;
    const float* mi = a.mi ? a.mi + r * a.n_in : nullptr;
    float dal[kTin];
    for (int t = 0; t < kTin; ++t) dal[t] = 0.0f;
    for (int j = lane; j < a.na2; j += 32) {
        const float dc = mi ? dX[j] * mi[j] : dX[j];
        for (int t = 0; t < kTin; ++t) dal[t] += dc * Ar[t * a.na2 + j];
    }
    for (int t = 0; t < kTin; ++t)
        for (int o = 16; o; o >>= 1) dal[t] += __shfl_xor_sync(0xffffffffu, dal[t], o);
    float al[kTin], de[kTin];
    float dot = 0.0f;
    for (int t = 0; t < kTin; ++t) {
        al[t] = a.alpha[r * kTin + t];
        dot += al[t] * dal[t];
    }
    float dps[ND];
    #pragma unroll
    for (int d = 0; d < ND; ++d) dps[d] = 0.0f;
    float dpre[kTin][ND];
    float dbo = 0.0f;
    for (int t = 0; t < kTin; ++t) {
        de[t] = al[t] * (dal[t] - dot);
        dbo += de[t];
        #pragma unroll
        for (int d = 0; d < ND; ++d) {
            const float hv = a.hid[(r * kTin + t) * ND + d];
            dpre[t][d] = de[t] * a.wo[d] * (1.0f - hv * hv);
            dps[d] += dpre[t][d];
        }
    }
    if (lane == 0) {
        float* ra = a.rowacc + r * (ND + 1);
        #pragma unroll
        for (int d = 0; d < ND; ++d) {
            float s = 0.0f;
            for (int t = 0; t < kTin; ++t) s += a.hid[(r * kTin + t) * ND + d] * de[t];
            ra[d] += s;
            a.DPs[r * ND + d] = dps[d];
        }
        ra[ND] += dbo;
        for (int t = 0; t < kTin; ++t)
            #pragma unroll
            for (int d = 0; d < ND; ++d) a.DPa[(r * kTin + t) * ND + d] += dpre[t][d];
    }
    for (int j = lane; j < a.na2; j += 32) a.dctx_out[r * a.na2 + j] = mi ? dX[j] * mi[j] : dX[j];
    const float* mr = a.mr ? a.mr + r * a.ns : nullptr;
    for (int j = lane; j < a.ns; j += 32) {
        float v = dX[a.na2 + j];
        if (mr) v *= mr[j];
        #pragma unroll
        for (int d = 0; d < ND; ++d) v += dps[d] * a.Ws[(long long)j * ND + d];
        a.dH[r * a.ns + j] = v;
    }
}

// dA[r][t] = sum_p alpha_p[r][t] dctx_p[r] + (sum_p dpre_p[r][t]) . Wa^T: the
// encoder activations' gradient from every decoder position at once (one pass
// instead of a read-modify-write of dA per position).  One warp per row.
struct AttnDA {
    int M, T, na2;
    const float* alpha;  // [T][M][7]
    const float* dctx;   // [T][M][na2]
    const float* DPa;    // [M][7][nd]
    const float* Wa;     // [na2][nd]
    float* dA;           // [M][7][na2]
};

template <int ND>
__global__ void k_attn_dA(AttnDA a) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= a.M) return;
    const long long r = warp, M = a.M;
    float dpa[kTin][ND];
    for (int t = 0; t < kTin; ++t)
#pragma unroll
        for (int d = 0; d < ND; ++d) dpa[t][d] = a.DPa[(r * kTin + t) * ND + d];
    for (int j = lane; j < a.na2; j += 32) {
        float acc[kTin];
        float wa[ND];
#pragma unroll
        for (int d = 0; d < ND; ++d) wa[d] = a.Wa[(long long)j * ND + d];
#pragma unroll
        for (int t = 0; t < kTin; ++t) {
            float v = 0.0f;
#pragma unroll
            for (int d = 0; d < ND; ++d) v += dpa[t][d] * wa[d];
            acc[t] = v;
        }
        for (int p = 0; p < a.T; ++p) {
            const float dc = a.dctx[((long long)p * M + r) * a.na2 + j];
            const float* al = a.alpha + ((long long)p * M + r) * kTin;
#pragma unroll
            for (int t = 0; t < kTin; ++t) acc[t] += al[t] * dc;
        }
#pragma unroll
        for (int t = 0; t < kTin; ++t) a.dA[(r * kTin + t) * a.na2 + j] = acc[t];
    }
}

// n_d (attention_dense_nodes) as a compile-time constant keeps the per-row
// energy terms in registers.
#define KST_ND_DISPATCH(kernel, Args)                                                      \
    inline bool launch_##kernel(int nd, const Args& a, unsigned grid, cudaStream_t s) {    \
        switch (nd) {                                                                      \
            case 1: kernel<1><<<grid, 256, 0, s>>>(a); return true;                        \
            case 2: kernel<2><<<grid, 256, 0, s>>>(a); return true;                        \
            case 3: kernel<3><<<grid, 256, 0, s>>>(a); return true;                        \
            case 4: kernel<4><<<grid, 256, 0, s>>>(a); return true;                        \
            case 5: kernel<5><<<grid, 256, 0, s>>>(a); return true;                        \
            case 6: kernel<6><<<grid, 256, 0, s>>>(a); return true;                        \
            case 7: kernel<7><<<grid, 256, 0, s>>>(a); return true;                        \
            case 8: kernel<8><<<grid, 256, 0, s>>>(a); return true;                        \
            default: return false;                                                         \
        }                                                                                  \
    }
KST_ND_DISPATCH(k_attn_fwd, AttnFwd)
KST_ND_DISPATCH(k_attn_bwd, AttnBwd)
KST_ND_DISPATCH(k_attn_dA, AttnDA)

// Head + cross entropy (dense_forward, cross_entropy_logits, sum_scaled 1/T;
// models.cpp:764-777), one warp per row: per-row loss (double), argmax match,
// dlogits = (softmax - onehot) / T and dh = dlogits . W^T.
struct HeadArgs {
    int M, ns, V, T, p;
    const float* h;      // [M][ns]
    const float* W;      // [ns][V]
    const float* b;      // [V]
    const int* tgt;      // [M][T]
    double* loss;        // [M] (this position)
    int* match;          // [M]
    float* dlog;         // [M][V]
    float* dh;           // [M][ns] or null (forward only)
};

__global__ void k_head(HeadArgs a) {
    extern __shared__ float sh[];
    const int warps = blockDim.x >> 5;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // W rows padded to V + 1 floats: lanes read rows j = lane + 32 i, so an odd row
    // stride keeps the 32 reads of a step in 32 different banks (stride V was a
    // V-way conflict)
    const int VS = a.V + 1;
    float* Wsm = sh;                          // ns * (V + 1)
    float* hrow = sh + a.ns * VS + w * (a.ns + 32);
    float* dsm = hrow + a.ns;                 // this warp's dlogits (32)
    for (int i = threadIdx.x; i < a.ns * a.V; i += blockDim.x) Wsm[(i / a.V) * VS + i % a.V] = a.W[i];
    __syncthreads();
    // persistent: the head weights are staged once per block, warps loop over rows
    for (long long r = (long long)blockIdx.x * warps + w; r < a.M; r += (long long)gridDim.x * warps) {
        for (int j = lane; j < a.ns; j += 32) hrow[j] = a.h[r * a.ns + j];
        __syncwarp();
        float lg = 0.0f;  // lane v holds logit v
        for (int v = 0; v < a.V; ++v) {
            float part = 0.0f;
            for (int j = lane; j < a.ns; j += 32) part += hrow[j] * Wsm[j * VS + v];
            for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
            if (lane == v) lg = part + a.b[v];
        }
        const bool act = lane < a.V;
        float mx = act ? lg : -INFINITY;
        for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        // argmax, lowest index on ties
        int am = (act && lg == mx) ? lane : 64;
        for (int o = 16; o; o >>= 1) am = min(am, __shfl_xor_sync(0xffffffffu, am, o));
        const float ex = act ? expf(lg - mx) : 0.0f;
        float s = ex;
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        const int t = a.tgt[r * a.T + a.p];
        const float lt = __shfl_sync(0xffffffffu, lg, t);
        if (lane == 0) {
            a.loss[r] = -((double)lt - (double)mx - log((double)s)) / a.T;
            a.match[r] = am == t ? 1 : 0;
        }
        const float d = act ? (ex / s - (lane == t ? 1.0f : 0.0f)) / (float)a.T : 0.0f;
        if (act) a.dlog[r * a.V + lane] = d;
        if (a.dh) {
            // dh = dlogits . W^T; the dlogits go through shared memory (the j loop's
            // trip count differs per lane, so no shuffles inside it)
            dsm[lane] = d;
            __syncwarp();
            for (int j = lane; j < a.ns; j += 32) {
                float v = 0.0f;
                for (int q = 0; q < a.V; ++q) v += dsm[q] * Wsm[j * VS + q];
                a.dh[r * a.ns + j] = v;
            }
        }
        __syncwarp();
    }
}

// Deterministic column sums: out[n] (+)= sum_r in[r * ld + n], two passes.
__global__ void k_colsum_partial(const float* in, long long R, int N, long long ld, int chunks, double* part) {
    const int n = blockIdx.x * 32 + threadIdx.x;
    const int c = blockIdx.y;
    __shared__ double red[8][33];
    double s = 0.0;
    if (n < N) {
        const long long per = (R + chunks - 1) / chunks;
        const long long r0 = c * per, r1 = min(R, r0 + per);
        for (long long r = r0 + threadIdx.y; r < r1; r += 8) s += in[r * ld + n];
    }
    red[threadIdx.y][threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.y == 0 && n < N) {
        double t = 0.0;
        for (int y = 0; y < 8; ++y) t += red[y][threadIdx.x];
        part[(long long)c * N + n] = t;
    }
}
// one warp per column: lanes stride over the chunks, fixed-order shuffle tree
__global__ void k_colsum_final(const double* part, int N, int chunks, float* out, int accumulate) {
    const int n = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (n >= N) return;
    double t = 0.0;
    for (int c = lane; c < chunks; c += 32) t += part[(long long)c * N + n];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) out[n] = accumulate ? out[n] + (float)t : (float)t;
}

// F16X3 operand splits: ksb::launch_absmax / ksb::launch_split_planes (ks_gemm16.cu)
using ksb::f16_scale_exp;

// Loss / match totals (double, fixed order).
__global__ void k_loss_total(const double* loss, const int* match, long long n, double* out_loss,
                             long long* out_match, int accumulate) {
    __shared__ double ls[256];
    __shared__ long long ms[256];
    double l = 0.0;
    long long m = 0;
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
        l += loss[i];
        m += match[i];
    }
    ls[threadIdx.x] = l;
    ms[threadIdx.x] = m;
    __syncthreads();
    for (int s = blockDim.x / 2; s; s >>= 1) {
        if (threadIdx.x < s) {
            ls[threadIdx.x] += ls[threadIdx.x + s];
            ms[threadIdx.x] += ms[threadIdx.x + s];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        if (out_loss) *out_loss = accumulate ? *out_loss + ls[0] : ls[0];
        if (out_match) *out_match = accumulate ? *out_match + ms[0] : ms[0];
    }
}

// Global norm of grads / batch (clip_global_norm, nn.cpp:286-297), two passes.
__global__ void k_sumsq(const float* g, long long n, double inv_b, double* part) {
    __shared__ double red[256];
    double s = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double v = (double)g[i] * inv_b;
        s += v * v;
    }
    red[threadIdx.x] = s;
    __syncthreads();
    for (int k = blockDim.x / 2; k; k >>= 1) {
        if (threadIdx.x < k) red[threadIdx.x] += red[threadIdx.x + k];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}
__global__ void k_norm_final(const double* part, int n, double* norm) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < n; ++i) s += part[i];
        *norm = sqrt(s);
    }
}

// adam_step (nn.cpp:262-284) on g / batch after the clip; fp64 per element.
__global__ void k_adam(float* p, float* m, float* v, const float* g, long long n, double inv_b, const double* norm,
                       double clip, double lr, double b1, double b2, double eps, double bc1, double bc2) {
    const double nn = *norm;
    const double scale = (nn <= clip || nn == 0.0) ? 1.0 : clip / nn;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double gi = (double)g[i] * inv_b * scale;
        const double mi = b1 * (double)m[i] + (1.0 - b1) * gi;
        const double vi = b2 * (double)v[i] + (1.0 - b2) * gi * gi;
        m[i] = (float)mi;
        v[i] = (float)vi;
        p[i] = (float)((double)p[i] - lr * (mi / bc1) / (sqrt(vi / bc2) + eps));
    }
}

}  // namespace kst

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
namespace {

using namespace kst;

// Allocation generation of the trainer whose API call is running on this thread
// (bumped on every (re)allocation of its buffers): captured training-step graphs
// bake buffer addresses, so a trainer's graph key includes ITS generation only --
// another trainer allocating (another GPU's thread, a second trainer in the same
// process) neither invalidates its graphs nor trips its post-capture check.
thread_local unsigned long long* tl_alloc_gen = nullptr;
struct GenScope {
    unsigned long long* prev;
    explicit GenScope(unsigned long long* g) : prev(tl_alloc_gen) { tl_alloc_gen = g; }
    ~GenScope() { tl_alloc_gen = prev; }
};

struct DBuf {
    void* p = nullptr;
    size_t bytes = 0;
    ~DBuf() {
        if (p) cudaFree(p);
    }
    cudaError_t ensure(size_t n) {
        if (n <= bytes) return cudaSuccess;
        if (tl_alloc_gen) ++*tl_alloc_gen;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        cudaError_t e = cudaMalloc(&p, n);
        if (e == cudaSuccess) bytes = n;
        return e;
    }
    template <class T>
    T* as() const { return reinterpret_cast<T*>(p); }
};

// One LSTM in the train layout: Wd [x_dense + H][4H], then Ws [S + 1][4H].
struct TLstm {
    std::string prefix;
    int x_dense = 0, S = 0, H = 0;
    long long off = 0;  // flat offset of Wd
    int Kd() const { return x_dense + H; }
    long long wd() const { return off; }
    long long ws() const { return off + (long long)Kd() * 4 * H; }
    long long size() const { return (long long)(Kd() + S + 1) * 4 * H; }
};

struct RefSeg {
    std::string name;
    long long numel;
    int lstm = -1;       // index into lstms, or -1: plain segment at `off`
    int gate = -1;       // 0..3 (input, forget, output, cand)
    bool bias = false;
    long long off = 0;
};

const char* kGateNames[4] = {"input", "forget", "output", "cand"};

}  // namespace

struct ks_trainer {
    int device = 0;
    int variant = 1;
    int T = 0;
    std::vector<int> vsize;
    int n_a = 0, n_s = 0, n_d = 0, e = 0;
    int d_in = 0, d_fb = 0;
    int in_off[kTin] = {};
    std::vector<int> fb_off;
    double dropout = 0.0, rdropout = 0.0;
    std::vector<TLstm> lstms;     // attn: pre.bwd, pre.fwd, post ; enc-dec: decoder, encoder
    int L_enc[2] = {-1, -1}, L_dec = -1;
    std::vector<RefSeg> segs;     // reference tensors in checkpoint order
    std::map<std::string, size_t> seg_of;
    long long off_attn_h = -1, off_attn_hb = -1, off_attn_o = -1, off_attn_ob = -1;
    std::vector<long long> off_head_w, off_head_b;
    long long nparams = 0;        // train-layout length (segments padded to 64 floats)
    long long nref = 0;           // reference parameter count (export / import order)
    DBuf params, adam_m, adam_v;
    long long adam_step = 0;
    cudaStream_t cur = nullptr;    // stream of the running batch (the GEMMs launch on it)
    int sms = 148;
    int cap_M = 0;
    // workspaces
    DBuf tok, tgt, idx, mi, mr, enc_slot, dec_slot, dec_val, enc_sm[2], dec_sm;
    DBuf Hx[2], Ce[2], Ze[2], dZe[2], A, U;
    DBuf Xd, Hs, Cd, Zd, dZd, alpha, hid, dlog, DHh, lossr, match;
    DBuf Xd16, Hx16[2];            // F16X3 planes of Xd / Hx written by their producers (hi, then lo)
    DBuf dXd, dH, dC, dA, Dctx, DPs, DPa, rowacc, dHe, dCe, part, norm, grads_tmp;
    DBuf res;                      // {loss sum, matches} of the last step / evaluate
    bool f16x3 = true;             // GEMMs as F16X3 on tcgen05 (default), else fp32 SIMT (KS_TRAIN_GEMM=fp32)
    DBuf scal;                     // F16X3: per-step max|x| slots and GEMM alphas; [2] = {0, 1} betas
    int scal_used = 0;
    int act_bound_bits = 0;        // the activation bound's float bits, written to its slot
    DBuf se;                       // {seed, epoch} of the current step (dropout masks)
    // CUDA graphs of whole ks_trainer_loss_grads batches on the trainer's own stream
    // (the caller's stream may be the legacy default stream, which cannot be captured)
    bool use_graphs = true;
    unsigned long long alloc_gen = 0;  // this trainer's buffer generation (GenScope)
    size_t head_attr = 0;              // k_head's dynamic-smem attribute set so far (on this trainer's device)
    cudaStream_t gs = nullptr;
    cudaEvent_t gev = nullptr;
    struct GraphEntry {
        std::vector<long long> key;
        cudaGraphExec_t exec = nullptr;
        long long launches = 0;
    };
    std::vector<GraphEntry> graphs;
    DBuf gpart, spart;             // split-K partials of the tensor-core / SIMT GEMMs
    // F16X3 operand planes of this batch: (source, rows, cols, ld) -> planes; weights and
    // operands several GEMMs share are split once per batch
    struct Planes {
        const __half* hi;
        const __half* lo;
        long long ld;
        const int* amax;
    };
    std::map<std::tuple<const float*, long long, long long, long long>, Planes> planes;
    std::vector<std::unique_ptr<DBuf>> plane_store;  // pool, reused batch after batch in call order
    size_t plane_used = 0;
    int n_in = 0;  // decoder input-mask width
    int vmax = 1;  // largest vocabulary (stride of the per-position dlogits blocks)
    long long launches = 0;
};

namespace {

#define KT_CUDA(call)                                                                              \
    do {                                                                                           \
        cudaError_t err_ = (call);                                                                 \
        if (err_ != cudaSuccess)                                                                   \
            return set_error(KS_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(err_));   \
    } while (0)

// fp32 SIMT GEMM (ks_gemm16.cu): exact fp32 FMAs, any transposes
ks_status gemm_simt(ks_trainer& t, bool ta, bool tb, long long M, long long N, long long K, const float* A,
                    long long lda, const float* B, long long ldb, float beta, float* C, long long ldc) {
    const int sp = ksb::sgemm_splits((int)M, (int)N, K, t.sms, ta);
    float* part = nullptr;
    if (sp > 1) {
        KT_CUDA(t.spart.ensure((size_t)sp * M * N * 4));
        part = t.spart.as<float>();
    }
    int n = 0;
    if (!ksb::launch_sgemm(ta, tb, (int)M, (int)N, K, A, lda, B, ldb, beta, C, ldc, part, t.sms, t.cur, &n))
        return set_error(KS_ERR_CUDA, "SIMT GEMM launch failed");
    t.launches += n;
    return KS_OK;
}


constexpr int kScalSlots = 4096;  // F16X3 per-step max|x| / alpha slots

// Row-major C[M x N] = op(A) op(B) + beta C on the trainer's stream.
// F16X3 (default): both operands split into fp16 hi/lo planes at power-of-two
// scales, in their own row-major layout (no transposes: the tcgen05 GEMM,
// ks_gemm16.cu, reads each operand K-major or MN-major), three MMA passes with
// fp32 accumulation, alpha = 2^-(eA+eB).  Weights (and operands two GEMMs of a
// step share, b_cache) are split once per batch: W serves the forward and dX.  a_amax / b_amax: device slots already
// holding max |A| / |B| (activations are tanh outputs times dropout scales; dZ
// maxima come fused from k_cell_bwd), so no max-reduction pass is needed.
// Narrow shapes (an output side under 16 / 128 columns: heads, attention) and
// KS_TRAIN_GEMM=fp32 run the fp32 SIMT GEMM.
ks_status gemm_rm(ks_trainer& t, bool ta, bool tb, long long M, long long N, long long K, const float* A,
                  long long lda, const float* B, long long ldb, float beta, float* C, long long ldc,
                  bool b_is_weight = false, const int* a_amax = nullptr, const int* b_amax = nullptr,
                  bool b_cache = false, const ks_trainer::Planes* apl = nullptr) {
    if (M == 0 || N == 0) return KS_OK;
    if (K == 0) return beta == 1.0f ? KS_OK : set_error(KS_ERR_SHAPE, "empty GEMM reduction");
    const bool narrow = b_cache ? (std::max(M, N) < 128 || std::min(M, N) < 16) : (M < 128 || N < 128);
    if (!t.f16x3 || narrow) return gemm_simt(t, ta, tb, M, N, K, A, lda, B, ldb, beta, C, ldc);
    if (beta != 0.0f && beta != 1.0f) return set_error(KS_ERR_PARAMETER, "F16X3 GEMM beta must be 0 or 1");

    cudaStream_t s = t.cur;
    int* slots = t.scal.as<int>();
    // hi / lo planes of a row-major [rows x cols] fp32 block (row stride ld), scale from
    // `amax` (a device slot already holding max|x|) or from a fresh max-reduction
    auto planes = [&](const float* src, long long rows, long long cols, long long ld, const int* amax, bool share,
                      ks_trainer::Planes& out) -> ks_status {
        const auto key = std::make_tuple(src, rows, cols, ld);
        if (share) {
            auto it = t.planes.find(key);
            if (it != t.planes.end()) {
                out = it->second;
                return KS_OK;
            }
        }
        if (!amax) {
            if (t.scal_used + 1 > kScalSlots) return set_error(KS_ERR_UNSUPPORTED, "too many GEMMs in one training step");
            int* slot = slots + t.scal_used++;
            ksb::launch_absmax(src, rows, cols, ld, slot, s);
            ++t.launches;
            amax = slot;
        }
        const long long ldo = (cols + 7) / 8 * 8;  // 16-byte rows (TMA)
        if (t.plane_used == t.plane_store.size()) t.plane_store.emplace_back(new DBuf());
        DBuf& buf = *t.plane_store[t.plane_used++];
        KT_CUDA(buf.ensure((size_t)rows * ldo * 2 * 2));
        __half* hi = buf.as<__half>();
        __half* lo = hi + rows * ldo;
        ksb::launch_split_planes(src, rows, cols, ld, hi, lo, ldo, amax, s);
        ++t.launches;
        out = {hi, lo, ldo, amax};
        if (share) t.planes.emplace(key, out);
        return KS_OK;
    };
    ks_status st;
    ks_trainer::Planes pa{}, pb{};
    // A: M x K (K-major) or, transposed, K x M (MN-major); B: K x N (MN-major) or N x K (K-major)
    if (apl)
        pa = *apl;  // written by the operand's producers
    else if ((st = planes(A, ta ? K : M, ta ? M : K, lda, a_amax, false, pa)))
        return st;
    if ((st = planes(B, tb ? N : K, tb ? K : N, ldb, b_amax, b_is_weight || b_cache, pb))) return st;
    const float* betap = reinterpret_cast<const float*>(slots + kScalSlots) + (beta == 0.0f ? 0 : 1);
    ksb::GemmF16Args g{pa.hi, pa.lo, pa.ld, ta ? 1 : 0, pb.hi, pb.lo, pb.ld, tb ? 0 : 1, (int)M, (int)N, K,
                       pa.amax, pb.amax, betap, C, ldc, nullptr, t.sms};
    const int sp = ksb::gemm16_splits((int)M, (int)N, K, t.sms);
    if (sp > 1) {
        KT_CUDA(t.gpart.ensure((size_t)sp * M * N * 4));
        g.part = t.gpart.as<float>();
    }
    int n = 0;
    if (!ksb::launch_gemm16(g, s, &n)) return set_error(KS_ERR_CUDA, "tensor-core GEMM launch failed");
    t.launches += n;
    return KS_OK;
}

ks_status colsum(ks_trainer& t, cudaStream_t s, const float* in, long long R, int N, long long ld, float* out,
                 bool accumulate) {
    const int chunks = (int)std::min<long long>(256, std::max<long long>(1, R / 64));
    KT_CUDA(t.part.ensure((size_t)chunks * N * 8));
    dim3 g((N + 31) / 32, chunks), b(32, 8);
    k_colsum_partial<<<g, b, 0, s>>>(in, R, N, ld, chunks, t.part.as<double>());
    k_colsum_final<<<(N + 7) / 8, 256, 0, s>>>(t.part.as<double>(), N, chunks, out, accumulate ? 1 : 0);
    t.launches += 2;
    return KS_OK;
}

inline unsigned blocks(long long n, int bs) { return (unsigned)((n + bs - 1) / bs); }

ks_status ensure_ws(ks_trainer& t, int M) {
    if (M <= t.cap_M) return KS_OK;
    const long long m = M;
    const int T = t.T;
    cudaError_t e = cudaSuccess;
#define TE(buf, n) do { if ((e = (buf).ensure((size_t)(n))) != cudaSuccess) goto fail; } while (0)
    TE(t.tok, m * 7 * 4);
    TE(t.tgt, m * T * 4);
    TE(t.idx, m * 8);
    TE(t.mi, m * std::max(1, t.n_in) * 4);
    TE(t.mr, m * std::max(1, t.lstms[t.L_dec].H) * 4);
    TE(t.enc_slot, 7 * m * 4);
    TE(t.dec_slot, T * m * 4);
    TE(t.dec_val, T * m * 4);
    TE(t.dec_sm, T * m * (t.lstms[t.L_dec].S + 1) * 4);
    for (int d = 0; d < 2; ++d) {
        if (t.L_enc[d] < 0) continue;
        const long long He = t.lstms[t.L_enc[d]].H;
        TE(t.enc_sm[d], 7 * m * (t.d_in + 1) * 4);
        TE(t.Hx[d], 8 * m * He * 4);
        TE(t.Hx16[d], 2 * 8 * m * ((He + 7) / 8 * 8) * 2);
        TE(t.Ce[d], 7 * m * He * 4);
        TE(t.Ze[d], 7 * m * 4 * He * 4);
        TE(t.dZe[d], 7 * m * 4 * He * 4);
    }
    {
        const TLstm& D = t.lstms[t.L_dec];
        const long long Hd = D.H, Kd = D.Kd();
        TE(t.Xd, T * m * Kd * 4);
        TE(t.Xd16, 2 * T * m * ((Kd + 7) / 8 * 8) * 2);
        TE(t.Hs, (T + 1) * m * Hd * 4);
        TE(t.Cd, T * m * Hd * 4);
        TE(t.Zd, T * m * 4 * Hd * 4);
        TE(t.dZd, T * m * 4 * Hd * 4);
        TE(t.dlog, T * m * t.vmax * 4);
        TE(t.DHh, T * m * Hd * 4);
        TE(t.lossr, T * m * 8);
        TE(t.match, T * m * 4);
        TE(t.dXd, m * Kd * 4);
        TE(t.dH, m * Hd * 4);
        TE(t.dC, m * Hd * 4);
        TE(t.dHe, m * std::max(1, t.variant == KS_VARIANT_ENC_DEC ? t.e : t.n_a) * 4);
        TE(t.dCe, m * std::max(1, t.variant == KS_VARIANT_ENC_DEC ? t.e : t.n_a) * 4);
    }
    if (t.variant != KS_VARIANT_ENC_DEC) {
        const long long na2 = 2LL * t.n_a;
        TE(t.A, m * 7 * na2 * 4);
        TE(t.U, m * 7 * t.n_d * 4);
        TE(t.alpha, T * m * 7 * 4);
        TE(t.hid, T * m * 7 * t.n_d * 4);
        TE(t.dA, m * 7 * na2 * 4);
        TE(t.Dctx, T * m * na2 * 4);
        TE(t.DPs, T * m * t.n_d * 4);
        TE(t.DPa, m * 7 * t.n_d * 4);
        TE(t.rowacc, m * (t.n_d + 1) * 4);
    }
    TE(t.norm, 8);
#undef TE
    t.cap_M = M;
    return KS_OK;
fail:
    return set_error(KS_ERR_CUDA, std::string("trainer workspace: ") + cudaGetErrorString(e));
}

// forward + (optional) backward of one batch already on the device.
ks_status run_batch(ks_trainer& t, int M, const int* d_tok, const int* d_tgt, const long long* d_idx,
                    long long dropout_epoch, unsigned long long seed, float* grads, bool accumulate,
                    double* d_loss, long long* d_match, cudaStream_t s) {
    ks_status st;
    if ((st = ensure_ws(t, M))) return st;
    t.cur = s;
    t.planes.clear();  // weights may have changed since the last call (Adam, import)
    t.plane_used = 0;
    // F16X3: fresh max|x| slots for this step's GEMMs; slot 0 bounds every activation
    // operand (LSTM outputs are tanh-bounded, times at most the dropout scale)
    int* act_amax = nullptr;
    auto new_slot = [&]() -> int* {
        if (!t.f16x3 || t.scal_used >= kScalSlots) return nullptr;  // null: the GEMM reduces itself
        return t.scal.as<int>() + t.scal_used++;
    };
    if (t.f16x3) {
        KT_CUDA(cudaMemsetAsync(t.scal.p, 0, (size_t)kScalSlots * 4, s));
        t.scal_used = 0;
        const float bound = (float)(1.0 / (1.0 - std::max(t.dropout, t.rdropout))) * 1.001f;
        std::memcpy(&t.act_bound_bits, &bound, 4);
        act_amax = new_slot();
        k_set_int<<<1, 1, 0, s>>>(act_amax, t.act_bound_bits);
        ++t.launches;
    }
    const int T = t.T;
    const long long m = M;
    const bool attn = t.variant != KS_VARIANT_ENC_DEC;
    const bool fbk = t.variant == KS_VARIANT_ATTN || t.variant == KS_VARIANT_ENC_DEC;
    TLstm& D = t.lstms[t.L_dec];
    const int Hd = D.H, Kd = D.Kd();
    float* P = t.params.as<float>();
    const bool drop = dropout_epoch >= 0 && (t.dropout != 0.0 || t.rdropout != 0.0);
    float* mi = drop ? t.mi.as<float>() : nullptr;
    float* mr = drop ? t.mr.as<float>() : nullptr;
    if (drop) {
        k_dropout_masks<<<blocks(m, 8), 256, 0, s>>>(M, t.se.as<unsigned long long>(), d_idx, 0, t.n_in, t.dropout, Hd,
                                                     t.rdropout, mi, mr);
        ++t.launches;
    }
    // slots
    SlotArgs sa{};
    sa.M = M;
    sa.T = T;
    sa.variant = t.variant;
    sa.tok = d_tok;
    sa.tgt = d_tgt;
    for (int f = 0; f < kTin; ++f) sa.in_off[f] = t.in_off[f];
    for (int p = 0; p < T; ++p) sa.fb_off[p] = t.fb_off[(size_t)p];
    sa.d_in = t.d_in;
    sa.d_fb = t.d_fb;
    sa.enc_dirs = attn ? 2 : 1;
    sa.dec_slots = D.S;
    sa.dec_mask_off = D.x_dense;
    sa.n_in = t.n_in;
    sa.mi = mi;
    sa.enc_slot = t.enc_slot.as<int>();
    sa.dec_slot = t.dec_slot.as<int>();
    sa.dec_val = t.dec_val.as<float>();
    sa.enc_sm[0] = t.enc_sm[0].as<float>();
    sa.enc_sm[1] = attn ? t.enc_sm[1].as<float>() : nullptr;
    sa.dec_sm = t.dec_sm.as<float>();
    k_slots<<<blocks((7 + T) * m, 256), 256, 0, s>>>(sa);
    ++t.launches;

    // ---------------------------------------------------------------- encoder
    const int dirs = attn ? 2 : 1;
    // F16X3 planes of the decoder operand X, written by its producers (attention: ctx,
    // the cells: h) at the activation bound's scale
    const TLstm& Dl = t.lstms[t.L_dec];
    const long long ldxq = (Dl.Kd() + 7) / 8 * 8;
    __half* xq_hi = t.f16x3 ? t.Xd16.as<__half>() : nullptr;
    __half* xq_lo = xq_hi ? xq_hi + (long long)T * m * ldxq : nullptr;
    for (int dir = 0; dir < dirs; ++dir) {
        const TLstm& L = t.lstms[t.L_enc[dir]];
        const int H = L.H;
        float* Hx = t.Hx[dir].as<float>();
        KT_CUDA(cudaMemsetAsync(Hx, 0, m * H * 4, s));
        // attn encoders: F16X3 planes of Hx (the recurrent operand) written by the cells
        const long long ldh16 = (H + 7) / 8 * 8;
        __half* hx_hi = (t.f16x3 && attn) ? t.Hx16[dir].as<__half>() : nullptr;
        __half* hx_lo = hx_hi ? hx_hi + 8LL * m * ldh16 : nullptr;
        if (hx_hi) {
            KT_CUDA(cudaMemsetAsync(hx_hi, 0, (size_t)m * ldh16 * 2, s));
            KT_CUDA(cudaMemsetAsync(hx_lo, 0, (size_t)m * ldh16 * 2, s));
        }
        for (int st_ = 0; st_ < kTin; ++st_) {
            const int tt = dir == 0 ? st_ : kTin - 1 - st_;
            float* Z = t.Ze[dir].as<float>() + (long long)st_ * m * 4 * H;
            const ks_trainer::Planes hp{hx_lo ? hx_hi + (long long)st_ * m * ldh16 : nullptr,
                                        hx_lo ? hx_lo + (long long)st_ * m * ldh16 : nullptr, ldh16, act_amax};
            if (st_ > 0 && (st = gemm_rm(t, false, false, m, 4LL * H, H, Hx + (long long)st_ * m * H, H,
                                         P + L.wd(), 4LL * H, 0.0f, Z, 4LL * H, true, act_amax, nullptr, false,
                                         hx_hi ? &hp : nullptr)))
                return st;
            CellFwd c{};
            c.M = M;
            c.H = H;
            c.S = L.S;
            c.Z = Z;
            c.zero_z = st_ == 0;
            c.Ws = P + L.ws();
            c.slot = t.enc_slot.as<int>() + (long long)tt * m;
            c.val = nullptr;
            c.c_prev = st_ == 0 ? nullptr : t.Ce[dir].as<float>() + (long long)(st_ - 1) * m * H;
            c.c_out = t.Ce[dir].as<float>() + (long long)st_ * m * H;
            if (attn) {
                c.h_out = t.A.as<float>() + (long long)tt * 2 * t.n_a + dir * t.n_a;
                c.ldh = 7LL * 2 * t.n_a;
                c.h_out2 = Hx + (long long)(st_ + 1) * m * H;
                c.ldh2 = H;
                if (hx_hi) {
                    c.q_hi = hx_hi + (long long)(st_ + 1) * m * ldh16;
                    c.q_lo = hx_lo + (long long)(st_ + 1) * m * ldh16;
                    c.ldq = ldh16;
                    c.qamax = act_amax;
                }
            } else {
                c.h_out = Hx + (long long)(st_ + 1) * m * H;
                c.ldh = H;
                if (st_ == kTin - 1) {  // enc-dec: the final h seeds the decoder operand X_0 (masked)
                    c.h_out2 = t.Xd.as<float>();
                    c.ldh2 = Kd;
                    c.mr = mr;
                    if (xq_hi) {
                        c.q_hi = xq_hi;
                        c.q_lo = xq_lo;
                        c.ldq = ldxq;
                        c.qamax = act_amax;
                    }
                }
            }
            launch_cell_fwd(c, s);
            ++t.launches;
        }
    }

    // ---------------------------------------------------------------- decoder
    float* Xd = t.Xd.as<float>();
    float* Hs = t.Hs.as<float>();
    const int na2 = 2 * t.n_a;
    float* Wh = attn ? P + t.off_attn_h : nullptr;   // [(ns + na2)][nd]: Ws rows, then Wa rows
    if (attn) {
        KT_CUDA(cudaMemsetAsync(Hs, 0, m * Hd * 4, s));
        // h part of X_0 = 0 (zero initial state)
        KT_CUDA(cudaMemset2DAsync(Xd + na2, (size_t)Kd * 4, 0, (size_t)Hd * 4, (size_t)m, s));
        if (xq_hi) {
            KT_CUDA(cudaMemset2DAsync(xq_hi + na2, (size_t)ldxq * 2, 0, (size_t)Hd * 2, (size_t)m, s));
            KT_CUDA(cudaMemset2DAsync(xq_lo + na2, (size_t)ldxq * 2, 0, (size_t)Hd * 2, (size_t)m, s));
        }
        if ((st = gemm_rm(t, false, false, 7 * m, t.n_d, na2, t.A.as<float>(), na2, Wh + (long long)t.n_s * t.n_d,
                          t.n_d, 0.0f, t.U.as<float>(), t.n_d)))
            return st;
    }
    for (int p = 0; p < T; ++p) {
        float* X = Xd + (long long)p * m * Kd;
        if (attn) {
            AttnFwd af{};
            af.M = M;
            af.na2 = na2;
            af.ns = t.n_s;
            af.nd = t.n_d;
            af.s = Hs + (long long)p * m * Hd;
            af.A = t.A.as<float>();
            af.U = t.U.as<float>();
            af.Ws = Wh;
            af.bh = P + t.off_attn_hb;
            af.wo = P + t.off_attn_o;
            af.bo = P + t.off_attn_ob;
            af.mi = mi;
            af.n_in = t.n_in;
            af.X = X;
            af.ldx = Kd;
            if (xq_hi) {
                af.x_hi = xq_hi + (long long)p * m * ldxq;
                af.x_lo = xq_lo + (long long)p * m * ldxq;
                af.ldxq = ldxq;
                af.qamax = act_amax;
            }
            af.alpha = t.alpha.as<float>() + (long long)p * m * 7;
            af.hid = t.hid.as<float>() + (long long)p * m * 7 * t.n_d;
            if (!launch_k_attn_fwd(t.n_d, af, blocks(m * 32, 256), s))
                return set_error(KS_ERR_UNSUPPORTED, "attention_dense_nodes outside 1..8");
            ++t.launches;
        }
        float* Z = t.Zd.as<float>() + (long long)p * m * 4 * Hd;
        const ks_trainer::Planes xp{xq_hi ? xq_hi + (long long)p * m * ldxq : nullptr,
                                    xq_hi ? xq_lo + (long long)p * m * ldxq : nullptr, ldxq, act_amax};
        if ((st = gemm_rm(t, false, false, m, 4LL * Hd, Kd, X, Kd, P + D.wd(), 4LL * Hd, 0.0f, Z, 4LL * Hd, true,
                          act_amax, nullptr, false, xq_hi ? &xp : nullptr)))
            return st;
        CellFwd c{};
        c.M = M;
        c.H = Hd;
        c.S = D.S;
        c.Z = Z;
        c.zero_z = 0;
        c.Ws = P + D.ws();
        c.slot = fbk ? t.dec_slot.as<int>() + (long long)p * m : nullptr;
        c.val = fbk ? t.dec_val.as<float>() + (long long)p * m : nullptr;
        c.c_prev = p == 0 ? (attn ? nullptr : t.Ce[0].as<float>() + 6 * m * t.e) : t.Cd.as<float>() + (long long)(p - 1) * m * Hd;
        c.c_out = t.Cd.as<float>() + (long long)p * m * Hd;
        c.h_out = Hs + (long long)(p + 1) * m * Hd;
        c.ldh = Hd;
        c.h_out2 = p + 1 < T ? Xd + (long long)(p + 1) * m * Kd + D.x_dense : nullptr;
        c.ldh2 = Kd;
        if (xq_hi && p + 1 < T) {
            c.q_hi = xq_hi + (long long)(p + 1) * m * ldxq + D.x_dense;
            c.q_lo = xq_lo + (long long)(p + 1) * m * ldxq + D.x_dense;
            c.ldq = ldxq;
            c.qamax = act_amax;
        }
        c.mr = mr;
        launch_cell_fwd(c, s);
        ++t.launches;
        // head + cross entropy
        HeadArgs ha{};
        ha.M = M;
        ha.ns = Hd;
        ha.V = t.vsize[(size_t)p];
        ha.T = T;
        ha.p = p;
        ha.h = Hs + (long long)(p + 1) * m * Hd;
        ha.W = P + t.off_head_w[(size_t)p];
        ha.b = P + t.off_head_b[(size_t)p];
        ha.tgt = d_tgt;
        ha.loss = t.lossr.as<double>() + (long long)p * m;
        ha.match = t.match.as<int>() + (long long)p * m;
        ha.dlog = t.dlog.as<float>() + (long long)p * m * t.vmax;
        ha.dh = grads ? t.DHh.as<float>() + (long long)p * m * Hd : nullptr;
        const int hw = 8;
        const size_t smem = ((size_t)Hd * (ha.V + 1) + (size_t)hw * (Hd + 32)) * 4;
        if (smem > 200 * 1024) return set_error(KS_ERR_UNSUPPORTED, "head too large for the head kernel");
        // function attributes are per device: each trainer sets it on its own device
        if (smem > 48 * 1024 && smem > t.head_attr) {
            KT_CUDA(cudaFuncSetAttribute(k_head, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            t.head_attr = smem;
        }
        k_head<<<(unsigned)std::min<long long>(blocks(m, hw), 148LL * 4), hw * 32, smem, s>>>(ha);
        ++t.launches;
    }
    k_loss_total<<<1, 256, 0, s>>>(t.lossr.as<double>(), t.match.as<int>(), (long long)T * m, d_loss, d_match,
                                  accumulate ? 1 : 0);
    ++t.launches;
    if (!grads) return KS_OK;

    // ---------------------------------------------------------------- backward
    float* G = grads;
    if (!accumulate) KT_CUDA(cudaMemsetAsync(G, 0, (size_t)t.nparams * 4, s));
    float* dH = t.dH.as<float>();
    float* dC = t.dC.as<float>();
    KT_CUDA(cudaMemsetAsync(dH, 0, m * Hd * 4, s));
    KT_CUDA(cudaMemsetAsync(dC, 0, m * Hd * 4, s));
    if (attn) {
        KT_CUDA(cudaMemsetAsync(t.DPa.p, 0, m * 7 * t.n_d * 4, s));
        KT_CUDA(cudaMemsetAsync(t.rowacc.p, 0, m * (t.n_d + 1) * 4, s));
    }
    int* dzd_amax = new_slot();  // max |dZ| over every position (the dW GEMM)
    for (int p = T - 1; p >= 0; --p) {
        float* dZ = t.dZd.as<float>() + (long long)p * m * 4 * Hd;
        int* dz_amax = new_slot();
        CellBwd cb{};
        cb.M = M;
        cb.H = Hd;
        cb.act = t.Zd.as<float>() + (long long)p * m * 4 * Hd;
        cb.c = t.Cd.as<float>() + (long long)p * m * Hd;
        cb.c_prev = p == 0 ? (attn ? nullptr : t.Ce[0].as<float>() + 6 * m * t.e) : t.Cd.as<float>() + (long long)(p - 1) * m * Hd;
        cb.dh1 = t.DHh.as<float>() + (long long)p * m * Hd;
        cb.ld1 = Hd;
        cb.dh2 = dH;
        cb.ld2 = Hd;
        cb.mask2 = attn ? nullptr : mr;  // enc-dec: dH is the raw dX of the next step's h rows
        cb.dc = dC;
        cb.dZ = dZ;
        cb.amax0 = dz_amax;
        cb.amax1 = dzd_amax;
        k_cell_bwd<<<std::min(blocks(m * Hd, 256), 148u * 8u), 256, 0, s>>>(cb);
        ++t.launches;
        // dX = dZ . Wd^T  -> [dctx | dh_rec]
        float* dX = t.dXd.as<float>();
        if ((st = gemm_rm(t, false, true, m, Kd, 4LL * Hd, dZ, 4LL * Hd, P + D.wd(), 4LL * Hd, 0.0f, dX, Kd, true,
                          dz_amax)))
            return st;
        if (attn) {
            AttnBwd ab{};
            ab.M = M;
            ab.na2 = na2;
            ab.ns = t.n_s;
            ab.nd = t.n_d;
            ab.dX = dX;
            ab.ldx = Kd;
            ab.mi = mi;
            ab.n_in = t.n_in;
            ab.mr = mr;
            ab.A = t.A.as<float>();
            ab.alpha = t.alpha.as<float>() + (long long)p * m * 7;
            ab.hid = t.hid.as<float>() + (long long)p * m * 7 * t.n_d;
            ab.Ws = Wh;
            ab.Wa = Wh + (long long)t.n_s * t.n_d;
            ab.wo = P + t.off_attn_o;
            ab.dctx_out = t.Dctx.as<float>() + (long long)p * m * na2;
            ab.dH = dH;
            ab.DPs = t.DPs.as<float>() + (long long)p * m * t.n_d;
            ab.DPa = t.DPa.as<float>();
            ab.rowacc = t.rowacc.as<float>();
            if (!launch_k_attn_bwd(t.n_d, ab, blocks(m * 32, 256), s))
                return set_error(KS_ERR_UNSUPPORTED, "attention_dense_nodes outside 1..8");
            ++t.launches;
        } else {
            // enc-dec: dH = dX (the recurrent rows) * mr, via the next cell_bwd's mask2
            KT_CUDA(cudaMemcpyAsync(dH, dX, m * Hd * 4, cudaMemcpyDeviceToDevice, s));
        }
    }
    // decoder weight gradients: one GEMM over all (position, row) pairs
    const ks_trainer::Planes xw{xq_hi, xq_lo, ldxq, act_amax};
    if ((st = gemm_rm(t, true, false, Kd, 4LL * Hd, (long long)T * m, Xd, Kd, t.dZd.as<float>(), 4LL * Hd, 1.0f,
                      G + D.wd(), 4LL * Hd, false, act_amax, dzd_amax, dzd_amax != nullptr, xq_hi ? &xw : nullptr)))
        return st;
    if ((st = gemm_rm(t, true, false, D.S + 1, 4LL * Hd, (long long)T * m, t.dec_sm.as<float>(), D.S + 1,
                      t.dZd.as<float>(), 4LL * Hd, 1.0f, G + D.ws(), 4LL * Hd, false, act_amax, dzd_amax,
                      dzd_amax != nullptr)))
        return st;
    for (int p = 0; p < T; ++p) {
        const int V = t.vsize[(size_t)p];
        const float* dl = t.dlog.as<float>() + (long long)p * m * t.vmax;
        if ((st = gemm_rm(t, true, false, Hd, V, m, Hs + (long long)(p + 1) * m * Hd, Hd, dl, V, 1.0f,
                          G + t.off_head_w[(size_t)p], V)))
            return st;
        if ((st = colsum(t, s, dl, m, V, V, G + t.off_head_b[(size_t)p], true))) return st;
    }
    if (attn) {
        // Ws rows: sum_p s_p^T DPs_p ; Wa rows: A^T DPa ; bh: colsum(DPa); attn.out: row sums
        if ((st = gemm_rm(t, true, false, t.n_s, t.n_d, (long long)T * m, Hs, Hd, t.DPs.as<float>(), t.n_d, 1.0f,
                          G + t.off_attn_h, t.n_d)))
            return st;
        if ((st = gemm_rm(t, true, false, na2, t.n_d, 7 * m, t.A.as<float>(), na2, t.DPa.as<float>(), t.n_d, 1.0f,
                          G + t.off_attn_h + (long long)t.n_s * t.n_d, t.n_d)))
            return st;
        if ((st = colsum(t, s, t.DPa.as<float>(), 7 * m, t.n_d, t.n_d, G + t.off_attn_hb, true))) return st;
        if ((st = colsum(t, s, t.rowacc.as<float>(), m, t.n_d, t.n_d + 1, G + t.off_attn_o, true))) return st;
        if ((st = colsum(t, s, t.rowacc.as<float>() + t.n_d, m, 1, t.n_d + 1, G + t.off_attn_ob, true))) return st;
        AttnDA da{};
        da.M = M;
        da.T = T;
        da.na2 = na2;
        da.alpha = t.alpha.as<float>();
        da.dctx = t.Dctx.as<float>();
        da.DPa = t.DPa.as<float>();
        da.Wa = Wh + (long long)t.n_s * t.n_d;
        da.dA = t.dA.as<float>();
        if (!launch_k_attn_dA(t.n_d, da, blocks(m * 32, 256), s))
            return set_error(KS_ERR_UNSUPPORTED, "attention_dense_nodes outside 1..8");
        ++t.launches;
    }
    // ---------------------------------------------------------------- encoder backward
    for (int dir = 0; dir < dirs; ++dir) {
        const TLstm& L = t.lstms[t.L_enc[dir]];
        const int H = L.H;
        float* dHe = t.dHe.as<float>();
        float* dCe = t.dCe.as<float>();
        if (attn) {
            KT_CUDA(cudaMemsetAsync(dHe, 0, m * H * 4, s));
            KT_CUDA(cudaMemsetAsync(dCe, 0, m * H * 4, s));
        } else {
            // enc-dec: the decoder's step-0 gradients flow into the encoder's final state
            KT_CUDA(cudaMemcpyAsync(dCe, dC, m * H * 4, cudaMemcpyDeviceToDevice, s));
        }
        int* dze_amax = new_slot();  // max |dZ| over the 7 steps (the dW GEMM)
        for (int st_ = kTin - 1; st_ >= 0; --st_) {
            const int tt = dir == 0 ? st_ : kTin - 1 - st_;
            float* dZ = t.dZe[dir].as<float>() + (long long)st_ * m * 4 * H;
            int* dz_amax = new_slot();
            CellBwd cb{};
            cb.M = M;
            cb.H = H;
            cb.act = t.Ze[dir].as<float>() + (long long)st_ * m * 4 * H;
            cb.c = t.Ce[dir].as<float>() + (long long)st_ * m * H;
            cb.c_prev = st_ == 0 ? nullptr : t.Ce[dir].as<float>() + (long long)(st_ - 1) * m * H;
            if (attn) {
                cb.dh1 = t.dA.as<float>() + (long long)tt * na2 + dir * t.n_a;
                cb.ld1 = 7LL * na2;
                cb.dh2 = dHe;
                cb.ld2 = H;
            } else {
                // enc-dec: the last step receives d(X_0) * mr from the decoder, earlier ones dHe
                cb.dh1 = nullptr;
                cb.dh2 = st_ == kTin - 1 ? dH : dHe;
                cb.ld2 = H;
                cb.mask2 = st_ == kTin - 1 ? mr : nullptr;
            }
            cb.dc = dCe;
            cb.dZ = dZ;
            cb.amax0 = dz_amax;
            cb.amax1 = dze_amax;
            k_cell_bwd<<<std::min(blocks(m * H, 256), 148u * 8u), 256, 0, s>>>(cb);
            ++t.launches;
            if (st_ > 0 && (st = gemm_rm(t, false, true, m, H, 4LL * H, dZ, 4LL * H, P + L.wd(), 4LL * H, 0.0f, dHe, H, true,
                                         dz_amax)))
                return st;
        }
        float* Hx = t.Hx[dir].as<float>();
        const long long ldh16 = (H + 7) / 8 * 8;
        __half* hx_hi = (t.f16x3 && attn) ? t.Hx16[dir].as<__half>() : nullptr;
        const ks_trainer::Planes hw{hx_hi, hx_hi ? hx_hi + 8LL * m * ldh16 : nullptr, ldh16, act_amax};
        if ((st = gemm_rm(t, true, false, H, 4LL * H, 7 * m, Hx, H, t.dZe[dir].as<float>(), 4LL * H, 1.0f,
                          G + L.wd(), 4LL * H, false, act_amax, dze_amax, dze_amax != nullptr, hx_hi ? &hw : nullptr)))
            return st;
        if ((st = gemm_rm(t, true, false, t.d_in + 1, 4LL * H, 7 * m, t.enc_sm[dir].as<float>(), t.d_in + 1,
                          t.dZe[dir].as<float>(), 4LL * H, 1.0f, G + L.ws(), 4LL * H, false, act_amax, dze_amax,
                          dze_amax != nullptr)))
            return st;
    }
    const cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return set_error(KS_ERR_CUDA, std::string("trainer kernels: ") + cudaGetErrorString(err));
    return KS_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------
namespace {

bool split_lstm_name(const std::string& n, std::string& prefix, int& gate, bool& bias) {
    const size_t dot = n.rfind('.');
    if (dot == std::string::npos) return false;
    const std::string tail = n.substr(dot + 1);
    prefix = n.substr(0, dot);
    for (int g = 0; g < 4; ++g) {
        if (tail == std::string("w_") + kGateNames[g]) { gate = g; bias = false; return true; }
        if (tail == std::string("b_") + kGateNames[g]) { gate = g; bias = true; return true; }
    }
    return false;
}

// reference row r of an LSTM weight ([x_dense | slots | h] x H) -> (Ws?, row)
inline long long lstm_elem(const TLstm& L, long long r, int g, long long j) {
    if (r < L.x_dense) return L.wd() + r * 4 * L.H + g * L.H + j;
    if (r < L.x_dense + L.S) return L.ws() + (r - L.x_dense) * 4 * L.H + g * L.H + j;
    return L.wd() + (L.x_dense + (r - L.x_dense - L.S)) * 4 * L.H + g * L.H + j;
}

// visits every reference element: fn(ref_flat_index, train_flat_index)
template <class F>
void for_each_elem(const ks_trainer& t, F fn) {
    long long ref = 0;
    for (const RefSeg& s : t.segs) {
        if (s.lstm < 0) {
            for (long long i = 0; i < s.numel; ++i) fn(ref + i, s.off + i);
        } else {
            const TLstm& L = t.lstms[(size_t)s.lstm];
            if (s.bias) {
                for (long long j = 0; j < L.H; ++j) fn(ref + j, L.ws() + (long long)L.S * 4 * L.H + s.gate * L.H + j);
            } else {
                const long long rows = s.numel / L.H;
                for (long long r = 0; r < rows; ++r)
                    for (long long j = 0; j < L.H; ++j) fn(ref + r * L.H + j, lstm_elem(L, r, s.gate, j));
            }
        }
        ref += s.numel;
    }
}

}  // namespace

extern "C" ks_status ks_trainer_create(const ks_model_desc* d, double dropout, double recurrent_dropout,
                                       int32_t device, ks_trainer** out) {
    if (!d || !out) return set_error(KS_ERR_PARAMETER, "null argument");
    *out = nullptr;
    if (d->variant != KS_VARIANT_ATTN && d->variant != KS_VARIANT_ATTN2 && d->variant != KS_VARIANT_ENC_DEC)
        return set_error(KS_ERR_UNSUPPORTED, "the B200 trainer implements the enc-dec, attn and attn-2 variants");
    if (dropout < 0.0 || dropout >= 1.0 || recurrent_dropout < 0.0 || recurrent_dropout >= 1.0)
        return set_error(KS_ERR_PARAMETER, "dropout rates must be in [0,1)");
    if (d->num_positions < 1 || d->num_positions > kMaxT)
        return set_error(KS_ERR_UNSUPPORTED, "1..16 output positions supported");
    if (d->attention_dense_nodes < 1 || d->attention_dense_nodes > kMaxNd)
        return set_error(KS_ERR_UNSUPPORTED, "1..8 attention dense nodes supported");
    if (cudaSetDevice(device) != cudaSuccess) return set_error(KS_ERR_CUDA, "cudaSetDevice failed");
    std::unique_ptr<ks_trainer> tr(new ks_trainer());
    ks_trainer& t = *tr;
    t.device = device;
    t.variant = d->variant;
    t.T = d->num_positions;
    t.n_a = d->pre_attention_size;
    t.n_s = d->post_attention_size;
    t.n_d = d->attention_dense_nodes;
    t.e = d->encoder_state_size;
    t.dropout = dropout;
    t.rdropout = recurrent_dropout;
    int off = 0;
    for (int f = 0; f < kTin; ++f) {
        t.in_off[f] = off;
        off += d->input_sizes[f];
    }
    t.d_in = off;
    off = 1;
    for (int p = 0; p < t.T; ++p) {
        const int v = d->vocab_sizes[p];
        if (v < 1 || v > 32) return set_error(KS_ERR_UNSUPPORTED, "vocabulary sizes 1..32 supported by the head kernel");
        t.vsize.push_back(v);
        t.vmax = std::max(t.vmax, v);
        t.fb_off.push_back(off);
        off += v;
    }
    t.d_fb = off;
    const bool attn = t.variant != KS_VARIANT_ENC_DEC;
    std::map<std::string, int> lstm_of;
    auto add_lstm = [&](const std::string& pfx, int xd, int S, int H) {
        TLstm L;
        L.prefix = pfx;
        L.x_dense = xd;
        L.S = S;
        L.H = H;
        lstm_of[pfx] = (int)t.lstms.size();
        t.lstms.push_back(L);
    };
    if (attn) {
        add_lstm("pre.fwd", 0, t.d_in, t.n_a);
        add_lstm("pre.bwd", 0, t.d_in, t.n_a);
        add_lstm("post", 2 * t.n_a, t.variant == KS_VARIANT_ATTN ? t.d_fb : 0, t.n_s);
        t.L_enc[0] = lstm_of["pre.fwd"];
        t.L_enc[1] = lstm_of["pre.bwd"];
        t.L_dec = lstm_of["post"];
        t.n_in = 2 * t.n_a + (t.variant == KS_VARIANT_ATTN ? t.d_fb : 0);
    } else {
        add_lstm("encoder", 0, t.d_in, t.e);
        add_lstm("decoder", 0, t.d_fb, t.e);
        t.L_enc[0] = lstm_of["encoder"];
        t.L_dec = lstm_of["decoder"];
        t.n_in = t.d_fb;
    }
    // layout, in the desc's tensor order (checkpoint order)
    // every segment starts 256-byte aligned: GEMM outputs land at segment starts and
    // the tensor-core kernels need aligned C (misaligned ones fall back to slow paths)
    auto pad_seg = [](long long x) { return (x + 63) / 64 * 64; };
    long long cursor = 0;
    std::vector<bool> placed(t.lstms.size(), false);
    std::vector<int> seen(t.lstms.size(), 0);
    t.off_head_w.assign((size_t)t.T, -1);
    t.off_head_b.assign((size_t)t.T, -1);
    for (int i = 0; i < d->num_tensors; ++i) {
        RefSeg sg;
        sg.name = d->tensor_names[i];
        sg.numel = d->tensor_numel[i];
        std::string pfx;
        int gate = -1;
        bool bias = false;
        if (split_lstm_name(sg.name, pfx, gate, bias) && lstm_of.count(pfx)) {
            const int li = lstm_of[pfx];
            TLstm& L = t.lstms[(size_t)li];
            const long long want = bias ? L.H : (long long)(L.x_dense + L.S + L.H) * L.H;
            if (sg.numel != want)
                return set_error(KS_ERR_SHAPE, "tensor " + sg.name + " has " + std::to_string(sg.numel) +
                                                   " elements, expected " + std::to_string(want));
            if (!placed[(size_t)li]) {
                L.off = cursor;
                cursor = pad_seg(cursor + L.size());
                placed[(size_t)li] = true;
            }
            sg.lstm = li;
            sg.gate = gate;
            sg.bias = bias;
            ++seen[(size_t)li];
        } else {
            sg.off = cursor;
            cursor = pad_seg(cursor + sg.numel);
            auto expect = [&](long long n) -> ks_status {
                return sg.numel == n ? KS_OK
                                     : set_error(KS_ERR_SHAPE, "tensor " + sg.name + " has " + std::to_string(sg.numel) +
                                                                   " elements, expected " + std::to_string(n));
            };
            ks_status st = KS_OK;
            if (sg.name == "attn.hidden.weights") { t.off_attn_h = sg.off; st = expect((long long)(t.n_s + 2 * t.n_a) * t.n_d); }
            else if (sg.name == "attn.hidden.bias") { t.off_attn_hb = sg.off; st = expect(t.n_d); }
            else if (sg.name == "attn.out.weights") { t.off_attn_o = sg.off; st = expect(t.n_d); }
            else if (sg.name == "attn.out.bias") { t.off_attn_ob = sg.off; st = expect(1); }
            else if (sg.name.rfind("head.", 0) == 0) {
                const int p = std::atoi(sg.name.c_str() + 5);
                const int hin = attn ? t.n_s : t.e;
                if (p < 0 || p >= t.T) return set_error(KS_ERR_STATE, "unexpected tensor " + sg.name);
                if (sg.name.size() > 8 && sg.name.compare(sg.name.size() - 8, 8, ".weights") == 0) {
                    t.off_head_w[(size_t)p] = sg.off;
                    st = expect((long long)hin * t.vsize[(size_t)p]);
                } else {
                    t.off_head_b[(size_t)p] = sg.off;
                    st = expect(t.vsize[(size_t)p]);
                }
            } else {
                return set_error(KS_ERR_STATE, "tensor " + sg.name + " does not belong to this variant");
            }
            if (st) return st;
        }
        t.seg_of[sg.name] = t.segs.size();
        t.segs.push_back(sg);
    }
    for (size_t li = 0; li < t.lstms.size(); ++li)
        if (seen[li] != 8) return set_error(KS_ERR_STATE, "model tensor set of '" + t.lstms[li].prefix + "' is incomplete");
    if (attn && (t.off_attn_h < 0 || t.off_attn_hb < 0 || t.off_attn_o < 0 || t.off_attn_ob < 0))
        return set_error(KS_ERR_STATE, "attention tensors missing");
    for (int p = 0; p < t.T; ++p)
        if (t.off_head_w[(size_t)p] < 0 || t.off_head_b[(size_t)p] < 0)
            return set_error(KS_ERR_STATE, "model tensor 'head." + std::to_string(p) + "' is missing");
    t.nparams = cursor;
    t.nref = 0;
    for (const RefSeg& sg : t.segs) t.nref += sg.numel;
    std::vector<float> host((size_t)cursor, 0.0f);
    std::vector<const float*> src((size_t)d->num_tensors);
    for (int i = 0; i < d->num_tensors; ++i) src[(size_t)i] = d->tensor_data[i];
    {
        // reference flat order = concatenation of the desc tensors
        std::vector<float> ref;
        ref.reserve((size_t)cursor);
        for (int i = 0; i < d->num_tensors; ++i) ref.insert(ref.end(), src[(size_t)i], src[(size_t)i] + d->tensor_numel[i]);
        for_each_elem(t, [&](long long r, long long q) { host[(size_t)q] = ref[(size_t)r]; });
    }
    cudaError_t e;
    if ((e = t.params.ensure((size_t)cursor * 4)) != cudaSuccess ||
        (e = t.adam_m.ensure((size_t)cursor * 4)) != cudaSuccess ||
        (e = t.adam_v.ensure((size_t)cursor * 4)) != cudaSuccess)
        return set_error(KS_ERR_CUDA, std::string("trainer allocation: ") + cudaGetErrorString(e));
    if (cudaMemcpy(t.params.p, host.data(), (size_t)cursor * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemset(t.adam_m.p, 0, (size_t)cursor * 4) != cudaSuccess ||
        cudaMemset(t.adam_v.p, 0, (size_t)cursor * 4) != cudaSuccess)
        return set_error(KS_ERR_CUDA, "trainer upload failed");
    {
        const char* g = std::getenv("KS_TRAIN_GEMM");
        // F16X3 on the tensor cores by default; KS_TRAIN_GEMM=fp32: the fp32 SIMT GEMM
        t.f16x3 = !(g && std::string(g) == "fp32");
        const float betas[2] = {0.0f, 1.0f};
        if (t.scal.ensure((size_t)(kScalSlots + 2) * 4) != cudaSuccess ||
            cudaMemcpy(t.scal.as<char>() + (size_t)kScalSlots * 4, betas, 8, cudaMemcpyHostToDevice) != cudaSuccess)
            return set_error(KS_ERR_CUDA, "trainer scale slots");
        cudaDeviceGetAttribute(&t.sms, cudaDevAttrMultiProcessorCount, t.device);
    }
    if (t.se.ensure(16) != cudaSuccess || cudaMemset(t.se.p, 0, 16) != cudaSuccess)
        return set_error(KS_ERR_CUDA, "trainer step scalars");
    {
        const char* kg = std::getenv("KS_GRAPHS");
        t.use_graphs = !(kg && kg[0] == '0');
        if (cudaStreamCreateWithFlags(&t.gs, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&t.gev, cudaEventDisableTiming) != cudaSuccess)
            return set_error(KS_ERR_CUDA, "trainer stream");
    }
    *out = tr.release();
    return KS_OK;
}

extern "C" ks_status ks_trainer_create_from_checkpoint(const char* path, int32_t device, ks_trainer** out) {
    ks_checkpoint* ck = nullptr;
    ks_status st = ks_checkpoint_load(path, &ck);
    if (st) return st;
    ksb_host::DescStore store;
    ks_model_desc d;
    st = ksb_host::desc_from_checkpoint(ck, store, d);
    const char* dr = ks_checkpoint_header(ck, "dropout");
    const char* rr = ks_checkpoint_header(ck, "recurrent_dropout");
    if (!st) st = ks_trainer_create(&d, dr ? std::atof(dr) : 0.0, rr ? std::atof(rr) : 0.0, device, out);
    ks_checkpoint_free(ck);
    return st;
}

extern "C" void ks_trainer_destroy(ks_trainer* t) {
    if (!t) return;
    cudaSetDevice(t->device);
    if (t->gs) cudaStreamSynchronize(t->gs);
    for (auto& g : t->graphs)
        if (g.exec) cudaGraphExecDestroy(g.exec);
    if (t->gev) cudaEventDestroy(t->gev);
    if (t->gs) cudaStreamDestroy(t->gs);
    delete t;
}

extern "C" int64_t ks_trainer_num_params(const ks_trainer* t) { return t ? t->nparams : 0; }
extern "C" int64_t ks_trainer_num_ref_params(const ks_trainer* t) { return t ? t->nref : 0; }
extern "C" int64_t ks_trainer_last_launch_count(const ks_trainer* t) { return t ? t->launches : 0; }

extern "C" ks_status ks_trainer_loss_grads(ks_trainer* t, const int32_t* d_tok, const int32_t* d_tgt,
                                           const int64_t* d_idx, int64_t B, int64_t dropout_epoch, uint64_t seed,
                                           float* d_grads, int32_t accumulate, double* d_loss_sum,
                                           int64_t* d_matches, void* stream) {
    GenScope gen_scope_(t ? &t->alloc_gen : nullptr);
    if (!t) return set_error(KS_ERR_PARAMETER, "null trainer");
    if (B < 0 || B > (1LL << 24)) return set_error(KS_ERR_PARAMETER, "batch size out of range");
    if (B == 0) return KS_OK;
    if (!d_tok || !d_tgt) return set_error(KS_ERR_PARAMETER, "null token buffer");
    cudaSetDevice(t->device);
    t->launches = 0;
    cudaStream_t user = reinterpret_cast<cudaStream_t>(stream);
    const long long* idx = reinterpret_cast<const long long*>(d_idx);
    long long* match = reinterpret_cast<long long*>(d_matches);
    ks_status st;
    if ((st = ensure_ws(*t, (int)B))) return st;
    if (!t->use_graphs) {
        k_set_u64x2<<<1, 1, 0, user>>>(t->se.as<unsigned long long>(), seed, (unsigned long long)dropout_epoch);
        t->launches = 1;
        return run_batch(*t, (int)B, d_tok, d_tgt, idx, dropout_epoch, seed, d_grads, accumulate != 0, d_loss_sum,
                         match, user);
    }
    // the whole batch (~250 launches) replays as one CUDA graph on the trainer stream;
    // seed / epoch are device values written just before it
    KT_CUDA(cudaEventRecord(t->gev, user));
    KT_CUDA(cudaStreamWaitEvent(t->gs, t->gev, 0));
    k_set_u64x2<<<1, 1, 0, t->gs>>>(t->se.as<unsigned long long>(), seed, (unsigned long long)dropout_epoch);
    // inputs staged into the trainer's own buffers: the graph key does not follow the
    // caller's (possibly per-step) input allocations
    KT_CUDA(cudaMemcpyAsync(t->tok.p, d_tok, (size_t)B * 7 * 4, cudaMemcpyDeviceToDevice, t->gs));
    KT_CUDA(cudaMemcpyAsync(t->tgt.p, d_tgt, (size_t)B * t->T * 4, cudaMemcpyDeviceToDevice, t->gs));
    if (idx) KT_CUDA(cudaMemcpyAsync(t->idx.p, idx, (size_t)B * 8, cudaMemcpyDeviceToDevice, t->gs));
    d_tok = t->tok.as<int32_t>();
    d_tgt = t->tgt.as<int32_t>();
    if (idx) idx = t->idx.as<long long>();
    auto P = [](const void* q) { return (long long)reinterpret_cast<uintptr_t>(q); };
    auto key_now = [&]() {
        return std::vector<long long>{B, P(d_tok), P(d_tgt), P(idx), P(d_grads), accumulate ? 1 : 0, P(d_loss_sum),
                                      P(match), dropout_epoch >= 0 ? 1 : 0,
                                      (long long)t->alloc_gen};
    };
    const std::vector<long long> key = key_now();
    ks_trainer::GraphEntry* hit = nullptr;
    for (auto& g : t->graphs)
        if (g.key == key) hit = &g;
    if (hit && hit->exec) {
        KT_CUDA(cudaGraphLaunch(hit->exec, t->gs));
        t->launches = 1 + hit->launches;
    } else if (!hit) {
        // first batch of this shape: plain launches, so every workspace reaches its size
        // (a buffer grown inside a capture would free memory already captured)
        t->launches = 1;
        st = run_batch(*t, (int)B, d_tok, d_tgt, idx, dropout_epoch, seed, d_grads, accumulate != 0, d_loss_sum,
                       match, t->gs);
        if (t->graphs.size() >= 8) {
            if (t->graphs.front().exec) cudaGraphExecDestroy(t->graphs.front().exec);
            t->graphs.erase(t->graphs.begin());
        }
        t->graphs.push_back({key_now(), nullptr, 0});
    } else {
        t->launches = 0;
        const bool began = cudaStreamBeginCapture(t->gs, cudaStreamCaptureModeRelaxed) == cudaSuccess;
        st = run_batch(*t, (int)B, d_tok, d_tgt, idx, dropout_epoch, seed, d_grads, accumulate != 0, d_loss_sum,
                       match, t->gs);
        cudaGraph_t graph = nullptr;
        const cudaError_t ce = began ? cudaStreamEndCapture(t->gs, &graph) : cudaErrorUnknown;
        cudaGraphExec_t exec = nullptr;
        const bool ok = began && !st && ce == cudaSuccess && graph &&
                        cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess;
        if (graph) cudaGraphDestroy(graph);
        if (!ok) {  // capture refused: this trainer runs plain launches from now on
            (void)cudaGetLastError();
            t->use_graphs = false;
            t->launches = 1;
            st = run_batch(*t, (int)B, d_tok, d_tgt, idx, dropout_epoch, seed, d_grads, accumulate != 0, d_loss_sum,
                           match, t->gs);
        } else {
            if (key_now() != key) {  // something was (re)allocated during the capture: do not keep it
                // drop this entry (re-captured on a later call under the new key);
                // graphs stay on
                cudaGraphExecDestroy(exec);
                hit->key = key_now();
                (void)cudaGetLastError();
                t->launches = 1;
                st = run_batch(*t, (int)B, d_tok, d_tgt, idx, dropout_epoch, seed, d_grads, accumulate != 0,
                               d_loss_sum, match, t->gs);
            } else {
                hit->exec = exec;
                hit->launches = t->launches;
                KT_CUDA(cudaGraphLaunch(exec, t->gs));
                t->launches += 1;
            }
        }
    }
    KT_CUDA(cudaEventRecord(t->gev, t->gs));
    KT_CUDA(cudaStreamWaitEvent(user, t->gev, 0));
    return st;
}

extern "C" ks_status ks_trainer_apply(ks_trainer* t, const float* d_grads, int64_t batch, double lr, double clip,
                                      void* stream) {
    GenScope gen_scope_(t ? &t->alloc_gen : nullptr);
    if (!t || !d_grads) return set_error(KS_ERR_PARAMETER, "null argument");
    if (batch < 1) return set_error(KS_ERR_PARAMETER, "batch must be >= 1");
    cudaSetDevice(t->device);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int nb = 592;
    KT_CUDA(t->part.ensure((size_t)nb * 8));
    KT_CUDA(t->norm.ensure(8));
    const double inv_b = 1.0 / (double)batch;
    k_sumsq<<<nb, 256, 0, s>>>(d_grads, t->nparams, inv_b, t->part.as<double>());
    k_norm_final<<<1, 32, 0, s>>>(t->part.as<double>(), nb, t->norm.as<double>());
    t->adam_step += 1;
    const double b1 = 0.9, b2 = 0.999, eps = 1e-8;  // AdamConfig (nn.hpp:96-101)
    const double bc1 = 1.0 - std::pow(b1, (double)t->adam_step);
    const double bc2 = 1.0 - std::pow(b2, (double)t->adam_step);
    k_adam<<<nb * 2, 256, 0, s>>>(t->params.as<float>(), t->adam_m.as<float>(), t->adam_v.as<float>(), d_grads,
                                   t->nparams, inv_b, t->norm.as<double>(), clip, lr, b1, b2, eps, bc1, bc2);
    t->launches += 3;
    const cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return set_error(KS_ERR_CUDA, std::string("apply: ") + cudaGetErrorString(err));
    return KS_OK;
}

extern "C" ks_status ks_trainer_step(ks_trainer* t, const int32_t* tok, const int32_t* tgt, const int64_t* idx,
                                     int64_t B, int64_t epoch, uint64_t seed, double lr, double clip,
                                     double* out_loss_sum, int64_t* out_matches) {
    GenScope gen_scope_(t ? &t->alloc_gen : nullptr);
    if (!t || !tok || !tgt) return set_error(KS_ERR_PARAMETER, "null argument");
    if (B < 1) return set_error(KS_ERR_PARAMETER, "batch must be >= 1");
    cudaSetDevice(t->device);
    ks_status st;
    if ((st = ensure_ws(*t, (int)B))) return st;
    if (!t->grads_tmp.p || t->grads_tmp.bytes < (size_t)t->nparams * 4)
        KT_CUDA(t->grads_tmp.ensure((size_t)t->nparams * 4));
    KT_CUDA(t->res.ensure(16));
    DBuf& res = t->res;
    cudaStream_t s = nullptr;
    KT_CUDA(cudaMemcpyAsync(t->tok.p, tok, (size_t)B * 7 * 4, cudaMemcpyHostToDevice, s));
    KT_CUDA(cudaMemcpyAsync(t->tgt.p, tgt, (size_t)B * t->T * 4, cudaMemcpyHostToDevice, s));
    if (idx) KT_CUDA(cudaMemcpyAsync(t->idx.p, idx, (size_t)B * 8, cudaMemcpyHostToDevice, s));
    k_set_u64x2<<<1, 1, 0, s>>>(t->se.as<unsigned long long>(), seed, (unsigned long long)epoch);
    t->launches = 1;
    if ((st = run_batch(*t, (int)B, t->tok.as<int>(), t->tgt.as<int>(), idx ? t->idx.as<long long>() : nullptr,
                        epoch, seed, t->grads_tmp.as<float>(), false, res.as<double>(),
                        reinterpret_cast<long long*>(res.as<char>() + 8), s)))
        return st;
    const long long l0 = t->launches;
    if ((st = ks_trainer_apply(t, t->grads_tmp.as<float>(), B, lr, clip, s))) return st;
    t->launches += l0;
    double hres[2];
    KT_CUDA(cudaMemcpyAsync(hres, res.p, 16, cudaMemcpyDeviceToHost, s));
    KT_CUDA(cudaStreamSynchronize(s));
    if (out_loss_sum) *out_loss_sum = hres[0];
    if (out_matches) std::memcpy(out_matches, &hres[1], 8);
    return KS_OK;
}

extern "C" ks_status ks_trainer_evaluate(ks_trainer* t, const int32_t* tok, const int32_t* tgt, int64_t B,
                                         double* out_loss_sum, int64_t* out_matches) {
    GenScope gen_scope_(t ? &t->alloc_gen : nullptr);
    if (!t || !tok || !tgt) return set_error(KS_ERR_PARAMETER, "null argument");
    if (B < 1) return set_error(KS_ERR_PARAMETER, "batch must be >= 1");
    cudaSetDevice(t->device);
    ks_status st;
    if ((st = ensure_ws(*t, (int)B))) return st;
    KT_CUDA(t->res.ensure(16));
    DBuf& res = t->res;
    cudaStream_t s = nullptr;
    KT_CUDA(cudaMemcpyAsync(t->tok.p, tok, (size_t)B * 7 * 4, cudaMemcpyHostToDevice, s));
    KT_CUDA(cudaMemcpyAsync(t->tgt.p, tgt, (size_t)B * t->T * 4, cudaMemcpyHostToDevice, s));
    t->launches = 0;
    if ((st = run_batch(*t, (int)B, t->tok.as<int>(), t->tgt.as<int>(), nullptr, -1, 0, nullptr, false,
                        res.as<double>(), reinterpret_cast<long long*>(res.as<char>() + 8), s)))
        return st;
    double hres[2];
    KT_CUDA(cudaMemcpyAsync(hres, res.p, 16, cudaMemcpyDeviceToHost, s));
    KT_CUDA(cudaStreamSynchronize(s));
    if (out_loss_sum) *out_loss_sum = hres[0];
    if (out_matches) std::memcpy(out_matches, &hres[1], 8);
    return KS_OK;
}

extern "C" ks_status ks_trainer_export(const ks_trainer* t, float* host_ref_flat) {
    if (!t || !host_ref_flat) return set_error(KS_ERR_PARAMETER, "null argument");
    cudaSetDevice(t->device);
    std::vector<float> host((size_t)t->nparams);
    KT_CUDA(cudaMemcpy(host.data(), t->params.p, (size_t)t->nparams * 4, cudaMemcpyDeviceToHost));
    for_each_elem(*t, [&](long long r, long long q) { host_ref_flat[r] = host[(size_t)q]; });
    return KS_OK;
}

extern "C" ks_status ks_trainer_import(ks_trainer* t, const float* host_ref_flat) {
    GenScope gen_scope_(t ? &t->alloc_gen : nullptr);
    if (!t || !host_ref_flat) return set_error(KS_ERR_PARAMETER, "null argument");
    cudaSetDevice(t->device);
    std::vector<float> host((size_t)t->nparams, 0.0f);
    for_each_elem(*t, [&](long long r, long long q) { host[(size_t)q] = host_ref_flat[r]; });
    KT_CUDA(cudaMemcpy(t->params.p, host.data(), (size_t)t->nparams * 4, cudaMemcpyHostToDevice));
    return KS_OK;
}

extern "C" ks_status ks_trainer_to_reference_layout(const ks_trainer* t, const float* host_train_flat,
                                                    float* host_ref_flat) {
    if (!t || !host_train_flat || !host_ref_flat) return set_error(KS_ERR_PARAMETER, "null argument");
    for_each_elem(*t, [&](long long r, long long q) { host_ref_flat[r] = host_train_flat[q]; });
    return KS_OK;
}
