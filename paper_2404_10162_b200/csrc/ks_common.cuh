// ks_common.cuh -- shared device-side types for the B200 beam-decode engine.
//
// HBM layout (one decode chunk of C configs, beam width k, padded hidden
// sizes NA = roundup(n_a, 64), NS = roundup(n_s, 64)):
//
//   tok      [C][7]          int32   input token ids
//   act      [C][7][2NA]     fp32    encoder activations a_t = [fwd_h ; bwd_h]
//   uatt     [C][7][n_d]     fp32    per-config attention term b_h + a_t.W_a
//   A        [C*k][2NA+NS]   fp32    (FP32 mode) decoder GEMM operand [ctx ; h_prev]
//   A_hi/lo  [C*k][2NA+NS]   fp16    (F16X3 / BF16 modes) the same operand, split
//   h, c     2 x [C*k][NS]   fp32    decoder state, ping-pong by position parity
//   beam     2 x {live u8, lp f64, key u64, parent i32, slot i32} per slot
//
// Rows of position p are r = b * H_p + j (H_p = static live-hypothesis bound,
// H_0 = 1, H_{p+1} = min(k, H_p * V_p)), so the GEMM M dimension carries no
// padding beyond the reference's own live counts in the unconstrained case.
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_bf16.h>

namespace ksb {

constexpr int kTin = 7;        // input fields n,c,h,w,k,y,x (problem.hpp:36-38)
constexpr int kMaxT = 16;      // output positions supported (builtin specs use <= 10)
constexpr int kMaxV = 32;      // vocabulary per position (lane-per-token in the beam kernel)
constexpr int kMaxNd = 8;      // attention dense nodes

// Per-position metadata passed by value to the beam kernel.
struct PosMeta {
    int T;
    int vsize[kMaxT];
    int value_offset[kMaxT];   // into the concatenated output-value table
    int fb_offset[kMaxT];      // feedback one-hot slot offset (GO = slot 0)
    int shift[kMaxT];          // packed-prefix key bit offset (position 0 in the MSBs)
    int bits[kMaxT];
};

// Device predicate program (see ks_pred in include/ks_b200.h).
struct DevPred {
    int kind;
    int full;
    int n_terms;
    int allowed_off;   // into the predicate byte table
    int terms_off;     // into the term arrays
    double budget;
    long long scale;
    long long limit;
};

// Fused LSTM step: gates = G[slot(r)] + A[r] . W, then the cell update
// (nn.cpp:88-128) with gate order i, f, o, cand.
struct LstmArgs {
    int M;             // rows
    int H;             // hidden units (padded, multiple of 64)
    int K;             // dense reduction length (multiple of 64, may be 0)
    // FP32 operand
    const float* A;
    long long lda;
    // split operand planes (row stride K)
    const __half* A_hi;
    const __half* A_lo;
    const float* W;    // FP32 mode: [K][4H], column u*4+g
    const float* G;    // [slots][4][H] = bias + one-hot weight row
    const int* slot_ptr;
    long long slot_stride;
    int slot_base;
    const float* c_prev;   // may be null -> zero state
    long long ldc_prev;
    const int* parent;     // row -> c_prev row; null -> identity; <0 -> zero state
    float* h_out;
    long long ldh;
    float* h_out2;         // optional second fp32 copy of h (hybrid: next operand + feature)
    long long ldh2;
    float* c_out;
    long long ldc;
    __half* hA_hi;         // optional split copy of h_out for the next GEMM
    __half* hA_lo;
    long long ldha;
    int ha_bf16;           // split copy as bf16 (BF16 mode) instead of fp16 hi/lo
    long long ldw;         // tensor-core W row stride in elements (0: K)
    int wcol;              // tensor-core W column offset (a K sub-range of the packed weight)
    long long ldah;        // tensor-core A-plane row stride in elements (0: K)
    // raw mode (the context projection P = a_t . W_ctx): no bias, no cell; the
    // pre-activations are stored TRANSPOSED and split for the alpha-block MMA:
    // pt_hi/lo[n][row], n = the tile's N index (gate-interleaved, = W row order)
    int raw;
    __half* pt_hi;
    __half* pt_lo;
    long long ldt;
    // alpha-block mode (projected context): the first kb_alpha K-blocks of the B
    // operand are P^T columns starting at 7 * b0(tile), b0 = first config of the
    // 128-row tile (rows_per_cfg rows per config); the A operand's first
    // 64*kb_alpha columns hold each row's alpha_t at 7 * (config - b0) + t
    int kb_alpha;
    int rows_per_cfg;
    int fan;               // > 1: row r is the shared parent of child rows r*fan .. r*fan+fan-1 (the
                           // epilogue adds each child's G[slot] and writes the children's h, c)
    int drop_pass;         // precision study only (KS_F16X2): 1 skips A_lo.W_hi, 2 skips A_hi.W_lo
    int alpha_tile;        // rows of the alpha-block layout tile: 128, or 256 for CTA-pair GEMMs
    const __half* PT_hi;   // P^T planes [4H][ldpt]
    const __half* PT_lo;
    long long ldpt;
    long long pt_rows;     // K extent of P^T (C * 7); reads beyond are zero-filled
    // compacted alpha-block positions (cp_M != null): rows are the DISTINCT live parents
    // of the position, *cp_M of them (M is the bound); row r belongs to config
    // cp_cfg[r] (the alpha-block tile spans configs cp_cfg[first row .. last row]), its
    // c_prev row is cp_prow[r], and its children are cp_child[cp_cstart[r] ..
    // + cp_ccount[r]) = {child row, slot, r, cp_prow[r]} (epilogue_compact); the
    // children of consecutive rows are consecutive entries
    const int* cp_M;
    const int* cp_cfg;
    const int* cp_prow;
    const int* cp_cstart;
    const int* cp_ccount;
    const int4* cp_child;
};

struct AttnArgs {
    int M;             // rows of this position
    int H_rows;        // rows per config at this position
    int NS;            // decoder hidden (padded)
    int NA2;           // 2 * NA
    int nd;
    const float* h_prev;   // previous-position h rows
    long long ldh;
    const int* parent;     // row -> h_prev row (<0 or null -> zero state)
    const float* act;      // [C][7][NA2]
    const float* uatt;     // [C][7][nd]
    const float* Ws;       // [NS][nd]  (attn.hidden rows for s_prev)
    const float* Wa;       // [NA2][nd] (attn.hidden rows for a_t), position 0 only
    const float* bh;       // [nd], position 0 only
    float* uatt_out;       // [C][7][nd] written at position 0
    const float* wo;       // [nd]
    float bo;
    float* A;              // FP32 operand out [M][a_ld]
    __half* A_hi;          // split operand out
    __half* A_lo;
    int split_mode;        // 0 fp32, 1 fp16 hi/lo (F16X3), 2 bf16 hi only (BF16)
    // alpha-block mode (kalpha > 0): instead of ctx, write the block-diagonal
    // alpha operand (kalpha columns, alpha_t at 7 * (config - b0(tile)) + t) and
    // h_prev after it; operand row stride kalpha + NS.  Classic: [ctx ; h_prev].
    int kalpha;
    int alpha_tile;        // rows of the GEMM tile the alpha block is laid out for (128 / 256)
    int alpha_sparse;      // alpha-block layout unchanged since the last position: write the 7 values only
    // compacted rows (LstmArgs::cp_M): row r = config cp_cfg[r], h_prev row cp_prow[r];
    // the alpha block follows the 128-row GEMM tile of r
    const int* cp_M;
    const int* cp_cfg;
    const int* cp_prow;
};

// Scales of the alpha-block MMA (F16X3): alpha in [0, 1] carries 2^12, P carries
// 2^4, so alpha.P accumulates at the same 2^16 as the 2^8-scaled h.W terms.
constexpr float kAlphaScale = 4096.0f;
// K-block of the tensor-core GEMM (fp16 elements per smem row): 64 -> 128-byte
// swizzle, 2 pipeline stages in F16X3 (32 -> 64-byte swizzle, 4 stages, is
// supported and parity-clean but measured 13% slower per launch).
constexpr int kTcBK = 64;
constexpr float kPScale = 16.0f;

struct BeamArgs {
    int B;
    int H_cur;
    int H_next;
    int pos;
    int k;
    int greedy;
    int final_step;
    int NS;
    const float* h;        // [B*H_cur][NS]
    const float* Wh;       // head weights [NS][V] (padded rows zero)
    const float* bh;       // [V]
    const unsigned char* live_cur;
    const double* lp_cur;
    const unsigned long long* key_cur;
    unsigned char* live_next;
    double* lp_next;
    unsigned long long* key_next;
    int* parent_next;
    int* slot_next;
    int* status;
    int* fail_pred;
    int* fail_step;
    const DevPred* preds;
    int n_preds;
    const unsigned char* pred_bytes;
    const int* term_pos;
    const double* term_w;
    const int* term_field;
    const long long* values;   // concatenated output values
    const long long* desc;     // [B][7] or null
    int* out_tok;              // [B][k][T]
    double* out_lp;            // [B][k]
    int* out_count;            // [B]
    int* out_fail_pred;
    int* out_fail_step;
    int* out_status;
    int cands_per_warp;        // smem capacity per warp (entries)
    const int* host_rej;       // [B*H_cur][V] first rejecting host predicate (or -1); may be null
    int h_per_config;          // hybrid: one feature row per config (static distributions)
    int n_values;              // staged-table sizes (shared memory)
    int n_terms;
    int n_bytes;
    // model_forward (models.cpp:495-514), greedy mode only: the fed-back token is
    // teacher[b][pos] instead of the argmax when teacher != null, and the position's
    // softmax distribution goes to out_dist[b][dist_off + v] (row stride dist_ld)
    const int* teacher;        // [B][T] or null
    double* out_dist;          // [B][dist_ld] or null
    int dist_ld;
    int dist_off;
};

// Hybrid variants' convolutional encoder arguments (hybrid_conv).
struct ConvArgs {
    int C;
    int n_conv;
    int f[8], k[8], s[8];
    const float* W[8];
    const float* b[8];
    int d_in;
    int in_offset[kTin];
    const int* tok;
    int F, FP, CP, K;
    int split_mode;
    __half* Ahi[4];  // [dir*2 + pingpong]
    __half* Alo[4];
    float* Af[4];
    int scratch_floats;  // per warp
};

// hybrid (layered) bi-LSTM 2 operands from bi-LSTM 1's sequence
struct HybPackArgs {
    const float* H1;   // [T][C][2CP]
    int C, T, CP;
    int split_mode;
    __half* Xhi[2];    // per direction [T][C][3CP]
    __half* Xlo[2];
    float* Xf[2];
};

// fp16 hi/lo split of an fp32 value, pre-scaled by 2^8 (exact) so that the
// residual of values down to ~5e-4 stays in the normal fp16 range:
//   x * 2^8 ~= hi + lo   (22 significant bits)
// Weights are split the same way at pack time, so one fp32 accumulator
// collects hi*hi + hi*lo + lo*hi = 2^16 * x.w and the epilogue scales by 2^-16.
constexpr float kSplitScale = 256.0f;
constexpr float kSplitUnscale = 1.0f / 65536.0f;

__device__ __forceinline__ void split_f16(float x, __half& hi, __half& lo) {
    const float xs = x * kSplitScale;
    hi = __float2half_rn(xs);
    lo = __float2half_rn(xs - __half2float(hi));   // residual exact in fp32
}

// split_f16 on two values at once: one paired fp32 multiply, packed f32->f16x2
// conversions and a paired subtract; bit-identical to two split_f16 calls.
__device__ __forceinline__ void split_f16x2(float x, float y, __half2& hi, __half2& lo) {
    const float2 s = __fmul2_rn(make_float2(x, y), make_float2(kSplitScale, kSplitScale));
    hi = __float22half2_rn(s);
    const float2 h = __half22float2(hi);
    lo = __float22half2_rn(__fadd2_rn(s, make_float2(-h.x, -h.y)));
}

// Same split at an explicit power-of-two scale (alpha-block operands).
__device__ __forceinline__ void split_f16s(float x, float scale, __half& hi, __half& lo) {
    const float xs = x * scale;
    hi = __float2half_rn(xs);
    lo = __float2half_rn(xs - __half2float(hi));
}

__device__ __forceinline__ void store_split_h(const LstmArgs& p, long long idx, float h) {
    if (p.ha_bf16) {
        reinterpret_cast<__nv_bfloat16*>(p.hA_hi)[idx] = __float2bfloat16_rn(h);
    } else {
        __half hi, lo;
        split_f16(h, hi, lo);
        p.hA_hi[idx] = hi;
        p.hA_lo[idx] = lo;
    }
}

// Function attributes (cudaFuncSetAttribute) are per device: `mask` records the
// devices a launcher has configured; returns true the first time for the current
// device (setting an attribute twice from racing threads is harmless).
inline bool first_on_device(std::atomic<unsigned long long>& mask) {
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    return (mask.fetch_or(bit) & bit) == 0;
}

}  // namespace ksb
