// ks_engine.cu -- the C-ABI (include/ks_b200.h): engine creation (weight
// packing into device layouts), workspace management, and the per-chunk
// decode schedule:
//
//   encoder   7 x lstm_step (both directions in one launch)   nn.cpp:130-165
//   uatt      a_t . W_a + b_h once per config                  models.cpp:265-281
//   for each output position p:                                decoding.cpp:45-94
//     attention_pack  rows B*H_p  -> [ctx ; h_prev] operand    models.cpp:466-478
//     lstm_step       gate GEMM + fused cell                   models.cpp:479-480
//     beam_step       head, log-softmax, predicates, top-k     models.cpp:490-492,
//                                                              decoding.cpp:49-93
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <atomic>
#include <mutex>
#include <thread>
#include <vector>

#include "ks_b200.h"
#include "ks_common.cuh"
#include "ks_internal.h"

namespace ksb {
__global__ void lstm_step_simt(LstmArgs a0, LstmArgs a1);
bool launch_lstm_k0(const LstmArgs& a0, const LstmArgs* a1, int sms, cudaStream_t s);
bool launch_attention(const AttnArgs& p, bool first, cudaStream_t s);
__global__ void beam_init(int B, unsigned char* live, double* lp, unsigned long long* key,
                          int* status, int* fail_pred, int* fail_step);
size_t beam_smem_bytes(int NS, int V, int warps, int cands_per_warp, size_t tables);
bool launch_beam(const BeamArgs& a, const PosMeta& m, int warps, size_t smem, int grid, cudaStream_t s);
bool launch_hybrid_conv(const ConvArgs& p, cudaStream_t s);
bool launch_hybrid_pack(const HybPackArgs& p, cudaStream_t s);
bool launch_topk_eval(const int* out_tok, const int* count, const int* truth, int B, int k, int T,
                      unsigned long long* pos_matches, unsigned long long* perfect, cudaStream_t s);
bool launch_split_rows(const float* src, long long n, __half* hi, __half* lo, int mode, cudaStream_t s);
// tensor-core gate GEMM (ks_gemm_tc.cu); returns false when the shape is not supported
bool launch_lstm_tc(const LstmArgs& a0, const LstmArgs* a1, int mode, const __half* W_hi0,
                    const __half* W_lo0, const __half* W_hi1, const __half* W_lo1,
                    cudaStream_t stream, int* launches, int units, bool pair);
}  // namespace ksb

using namespace ksb;

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
namespace {
thread_local std::string g_msg;
thread_local std::string g_field;
}  // namespace

namespace ksb_host {
ks_status set_error(ks_status code, const std::string& msg, const std::string& field) {
    g_msg = msg;
    g_field = field;
    return code;
}
}  // namespace ksb_host
using ksb_host::set_error;

extern "C" const char* ks_last_error(void) { return g_msg.c_str(); }
extern "C" const char* ks_last_error_field(void) { return g_field.c_str(); }

#define KS_CUDA(call)                                                                   \
    do {                                                                                \
        cudaError_t err_ = (call);                                                      \
        if (err_ != cudaSuccess)                                                        \
            return set_error(KS_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(err_)); \
    } while (0)

namespace {

int round_up(int x, int m) { return (x + m - 1) / m * m; }
constexpr int SB_M_HOST = 64;

// bumped on every device (re)allocation: captured decode graphs bake buffer
// addresses into their kernel parameters and are re-captured when it moves
std::atomic<unsigned long long> g_alloc_gen{0};

struct DevMem {
    void* p = nullptr;
    size_t bytes = 0;
    ~DevMem() {
        if (p) cudaFree(p);
    }
    cudaError_t ensure(size_t n) {
        if (n <= bytes) return cudaSuccess;
        g_alloc_gen.fetch_add(1);
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

struct HostMem {
    void* p = nullptr;
    size_t bytes = 0;
    ~HostMem() {
        if (p) cudaFreeHost(p);
    }
    cudaError_t ensure(size_t n) {
        if (n <= bytes) return cudaSuccess;
        if (p) cudaFreeHost(p);
        p = nullptr;
        bytes = 0;
        cudaError_t e = cudaMallocHost(&p, n);
        if (e == cudaSuccess) bytes = n;
        return e;
    }
    template <class T>
    T* as() const { return reinterpret_cast<T*>(p); }
};

// One packed LSTM cell on the device.
struct DevLstm {
    int H = 0, K = 0, slots = 0;
    DevMem W;       // FP32: [K][4H] (u*4+g)
    DevMem Whi;     // TC: [4H][K] gate-interleaved per 64-unit tile
    DevMem Wlo;
    DevMem Whi32;   // the same planes interleaved per 32-unit tile (small batches)
    DevMem Wlo32;
    DevMem G;       // [slots][4][H]
};

}  // namespace

struct ks_engine {
    int device = 0;
    int precision = KS_PREC_F16X3;
    int variant = 1;
    int n_a = 0, n_s = 0, n_d = 0, e = 0;
    int NA = 0, NS = 0, NE = 0;
    int T = 0;
    int d_in = 0, d_fb = 0;
    std::vector<int> vsize, in_sizes, in_offset;
    std::vector<int64_t> in_values, out_values;
    PosMeta meta{};
    DevLstm enc[2], dec;
    DevMem attWs, attWa, attBh, attWo;
    float attBo = 0.0f;
    std::vector<std::unique_ptr<DevMem>> headW, headB;
    DevMem values;
    // workspace
    int64_t chunk = 65536;
    DevMem tok, desc, act, uatt, encc, encA, Abuf, Ahi, Alo, hbuf, cbuf;
    DevMem live[2], lp[2], key[2], parent[2], slot[2], status, fpred, fstep;
    DevMem otok, olp, ocount, ostatus, ofpred, ofstep;
    DevMem preds, pbytes, tpos, tw, tfield;
    DevMem hrej;                  // host-hook rejections [C*k][Vmax]
    DevMem truth, evalc;          // topk_metrics: truths [C][T], counters [T + 1]
    HostMem h_in, h_out, hk_keys, hk_live, hk_rej;
    // chunk pipeline (decode_chunks): two sets of chunk I/O buffers; chunk i decodes
    // from / into set i & 1 on `stream` while the results of chunk i - 1 leave on
    // `copy_stream` and are unpacked on the host
    struct ChunkIO {
        DevMem tok, desc, otok, olp, ocount, ostatus, ofpred, ofstep;
        HostMem h_in, h_out;
        cudaEvent_t dec_done = nullptr, copy_done = nullptr;
    } io[2];
    cudaStream_t copy_stream = nullptr;
    cudaStream_t stream = nullptr;
    int64_t launches = 0;
    int beam_smem_max = 0;
    // profiling of the gate GEMM launches
    bool prof = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_ev;
    std::vector<double> prof_flops, prof_exec;
    double prof_ms = 0.0, prof_useful = 0.0;
    std::vector<std::pair<double, double>> prof_each;  // per GEMM launch: (ms, useful FLOPs)
    std::vector<double> prof_each_exec;                // per GEMM launch: MMA FLOPs issued
    int64_t prof_n = 0;
    int tc_units = 64;
    // hybrid-2 (models.cpp:296-371, 409-425)
    int cell = 0, CP = 0, F = 0, FP = 0;
    std::vector<int> conv_f, conv_k, conv_s;
    std::vector<std::unique_ptr<DevMem>> convW, convB;
    int conv_scratch = 0;
    DevLstm hb1[2], hb2[2];
    DevMem hybA, hybAf, hybC, hybH, feat;
    std::mutex mu;                // calls share the workspace: one decode at a time per engine
    // predicate tables last uploaded (identical tables are not re-uploaded; a change
    // waits for the engine stream so in-flight decodes never see a half-written table)
    std::vector<unsigned char> pred_blob;
    // CUDA graphs of whole single-chunk decodes, keyed by everything their kernel
    // parameters bake in (KS_GRAPHS=0 disables)
    bool use_graphs = true;
    bool pt_valid = false;  // the workspace's P^T belongs to the last encoded chunk
    // launches without an alpha block (encoder, context projection, position 0) run on
    // CTA pairs (M = 256 tcgen05.mma.cta_group::2: half the B operand traffic per SM);
    // alpha-block positions keep single-CTA tiles (a 256-row tile would double the
    // alpha columns) and so does the epilogue-bound position-1 fan-out
    bool pair_auto = true;
    struct GraphEntry {
        std::vector<long long> key;
        cudaGraphExec_t exec = nullptr;
        int64_t launches = 0;
    };
    std::vector<GraphEntry> graphs;
    ~ks_engine() {
        for (auto& g : graphs)
            if (g.exec) cudaGraphExecDestroy(g.exec);
        for (auto& b : io) {
            if (b.dec_done) cudaEventDestroy(b.dec_done);
            if (b.copy_done) cudaEventDestroy(b.copy_done);
        }
        if (copy_stream) cudaStreamDestroy(copy_stream);
    }
    // model_forward (ks_forward_batch): set for the duration of that call only
    const int* fw_teacher = nullptr;  // device [C][T] teacher tokens of the chunk, or null (argmax)
    double* fw_dist = nullptr;        // device [C][sum V] distributions of the chunk
    int fw_ld = 0;
    DevMem fwt, fwd;
    bool layered = false;         // hybrid: bi-LSTM 2 runs over bi-LSTM 1's sequence (not seeded)
    DevMem hybH1, hybX2;          // layered: H1 [T][C][2CP] fp32; bi-LSTM 2 operands per dir and step
    int num_sms = 148;
    // projected context (attn / attn-2, tensor-core modes): ctx . W_ctx =
    // sum_t alpha_t (a_t . W_ctx).  P = a_t . W_ctx is computed once per config
    // (stored transposed, split: Pt [2][4NS][ldt]); from position 1 on the
    // decoder GEMM contracts [alpha block | h_prev] against [P^T | W_h]
    bool ctxproj = false;
    bool ctxproj_force = false;   // KS_CTXPROJ=force: alpha blocks even where wider than ctx (tests)
    DevMem Pt, actA;
    DevMem encp;  // shared-prefix encoder tables of the current chunk
    // compacted alpha-block positions: the GEMM and attention run on each
    // config's distinct live parents, the epilogue writes their children
    // (KS_COMPACT=0 disables)
    bool compact = true;
    bool compact_pos1 = false;   // KS_COMPACT_POS1=1: position 1 compacted too instead of the fan-out
                                 // epilogue (measured slower: 1.37 vs 1.12 ms at cfg2)
    bool debug_parents = false;  // KS_DEBUG_PARENTS=1: print distinct parents per position (not with graphs)
    DevMem dbg;
    DevMem cpbuf;  // [C] counts, [C + 1] bases (last = rows), [R] cfg, prow, cstart, ccount, [R] int2 children
    // KS_TC_PAIR=1: gate GEMMs on CTA pairs (M = 256 tiles, tcgen05 cta_group::2)
    bool pair = false;
    // N-tile width of the current chunk's gate GEMMs: tc_units, or 32 when 64-unit
    // tiles would leave SMs idle (small batches; needs the 32-unit weight planes)
    int units_now = 64;
    // shared-prefix encoder (attn / attn-2 with the a_t operand planes): the state of
    // encoder step s of a direction depends only on the first s+1 input fields that
    // direction reads.  When a chunk holds more configs than a step has token
    // prefixes, the step runs once per PREFIX (all of them, a static shape) instead of
    // once per config -- one gate-GEMM launch over the step's prefixes, the parents'
    // split h replicated as its A operand -- and a gather hands every config its
    // states (KS_ENC_PREFIX=0 disables)
    struct EncTable {
        int S = -1;                 // steps 0..S can run per prefix (-1: none)
        int order[7] = {};          // field read at step j (fwd t = j, bwd t = 6 - j)
        int size[7] = {};           // |field| of step j
        long long R[7] = {};        // prefixes of step j: prod_{i<=j} size[i]
        long long off[7] = {};      // first row of step j in the prefix tables (sum_{i<j} R[i])
        DevMem digits;              // [2][sum R]: step j's new digit of prefix r (r % size[j]) at
                                    // off[j] + r, then its parent prefix (r / size[j])
        long long total = 0;        // sum R
    };
    // chunks below this many configs encode per config: their launches are latency-bound,
    // so the prefix steps' extra launches (replicate, gather) cost more than they save
    int64_t prefix_min = 16384;
    EncTable etab[2];
    bool pair_now() const { return pair && units_now == 64; }
    bool proj_at(int pos, int H) const {
        return ctxproj && pos > 0 && (ctxproj_force || alpha_cols_of(H) < 2 * NA);
    }
    // Alpha-block columns for TR-row tiles of H rows per config: TR % H == 0 ->
    // every tile holds TR / H whole configs; otherwise up to (TR - 1) / H + 2
    // (partial configs at both ends); 7 columns each, plus up to 7 columns of
    // 8-alignment of the first (tile_k, ks_gemm_tc.cu), rounded to the K-block.
    static int alpha_cols_for(int TR, int H) {
        const int cfgs = TR % H == 0 ? TR / H : (TR - 1) / H + 2;
        return (7 * cfgs + 7 + kTcBK - 1) / kTcBK * kTcBK;
    }
    // Rows per alpha-block GEMM tile: a CTA pair's 256, else 128 or the largest
    // multiple of H below it (config-aligned: e.g. 125 rows = 25 configs at beam 5
    // need 3 alpha K-blocks instead of 4), whichever contracts fewer columns per row.
    int alpha_tile_of(int H) const {
        if (pair_now()) return 256;
        const int ra = H <= 128 ? 128 / H * H : 128;
        const double plain = (NS + alpha_cols_for(128, H)) / 128.0;
        const double aligned = (NS + alpha_cols_for(ra, H)) / (double)ra;
        return aligned < plain ? ra : 128;
    }
    int alpha_cols_of(int H) const { return alpha_cols_for(alpha_tile_of(H), H); }
};

// Columns of the alpha block for rows_per_cfg rows per config: a TR-row tile
// (128, or 256 for CTA pairs) spans at most (TR - 1) / H + 2 configs, 7 columns
// each, plus up to 7 columns of 8-alignment of the first (tile_k,
// ks_gemm_tc.cu), rounded to the K-block.

namespace {

// ---------------------------------------------------------------------------
// weight packing
// ---------------------------------------------------------------------------
struct HostTensors {
    std::map<std::string, std::pair<const float*, int>> m;
    const float* get(const std::string& n, int numel_expect, std::string& err) const {
        auto it = m.find(n);
        if (it == m.end()) {
            err = "model tensor '" + n + "' is missing";
            return nullptr;
        }
        if (numel_expect >= 0 && it->second.second != numel_expect) {
            err = "tensor '" + n + "' has " + std::to_string(it->second.second) + " values, expected " +
                  std::to_string(numel_expect);
            return nullptr;
        }
        return it->second.first;
    }
};

// Packs a reference LSTM cell (4 gate matrices (rows x H) + 4 biases) whose
// rows split into a dense part (device k -> reference row, -1 = zero) and a
// one-hot part (slot -> reference row, -1 = bias only).
ks_status pack_lstm(const HostTensors& ht, const std::string& prefix, int rows, int H, int Hp,
                    const std::vector<int>& dense_rows, const std::vector<int>& slot_rows,
                    DevLstm& out, int precision, int units) {
    static const char* gates[4] = {"input", "forget", "output", "cand"};
    std::string err;
    const float* W[4];
    const float* Bv[4];
    for (int g = 0; g < 4; ++g) {
        W[g] = ht.get(prefix + ".w_" + gates[g], rows * H, err);
        if (!W[g]) return set_error(KS_ERR_STATE, err);
        Bv[g] = ht.get(prefix + ".b_" + gates[g], H, err);
        if (!Bv[g]) return set_error(KS_ERR_STATE, err);
    }
    const int K = (int)dense_rows.size();
    const int S = (int)slot_rows.size();
    out.H = Hp;
    out.K = K;
    out.slots = S;
    std::vector<float> Wf((size_t)K * 4 * Hp, 0.0f);
    std::vector<__half> Whi((size_t)4 * Hp * K), Wlo((size_t)4 * Hp * K);
    std::vector<float> G((size_t)S * 4 * Hp, 0.0f);
    for (int k = 0; k < K; ++k) {
        const int r = dense_rows[(size_t)k];
        for (int u = 0; u < Hp; ++u)
            for (int g = 0; g < 4; ++g) {
                const float w = (r >= 0 && u < H) ? W[g][(size_t)r * H + u] : 0.0f;
                if (std::fabs(w) > 200.0f)
                    return set_error(KS_ERR_UNSUPPORTED, "weight magnitude exceeds the fp16 split range");
                Wf[(size_t)k * 4 * Hp + u * 4 + g] = w;
                // tensor-core layout: N index n = blk*4U + g*U + u%U (blk = u/U), K-major
                const size_t n = (size_t)(u / units) * 4 * units + (size_t)g * units + (u % units);
                if (precision == KS_PREC_BF16) {
                    const __nv_bfloat16 hb = __float2bfloat16_rn(w);
                    std::memcpy(&Whi[n * K + k], &hb, 2);
                    Wlo[n * K + k] = __float2half_rn(0.0f);
                } else {  // same 2^8-scaled split as split_f16 (ks_common.cuh)
                    const float ws = w * 256.0f;
                    const __half hi = __float2half_rn(ws);
                    Whi[n * K + k] = hi;
                    Wlo[n * K + k] = __float2half_rn(ws - __half2float(hi));
                }
            }
    }
    for (int s = 0; s < S; ++s) {
        const int r = slot_rows[(size_t)s];
        for (int g = 0; g < 4; ++g)
            for (int u = 0; u < H; ++u) {
                float v = Bv[g][u];
                if (r >= 0) v += W[g][(size_t)r * H + u];
                G[(size_t)s * 4 * Hp + (size_t)g * Hp + u] = v;
            }
    }
    cudaError_t e = cudaSuccess;
    if (K > 0) {
        if ((e = out.W.ensure(Wf.size() * 4)) != cudaSuccess) goto fail;
        if ((e = cudaMemcpy(out.W.p, Wf.data(), Wf.size() * 4, cudaMemcpyHostToDevice))) goto fail;
        if ((e = out.Whi.ensure(Whi.size() * 2)) != cudaSuccess) goto fail;
        if ((e = out.Wlo.ensure(Wlo.size() * 2)) != cudaSuccess) goto fail;
        if ((e = cudaMemcpy(out.Whi.p, Whi.data(), Whi.size() * 2, cudaMemcpyHostToDevice))) goto fail;
        if ((e = cudaMemcpy(out.Wlo.p, Wlo.data(), Wlo.size() * 2, cudaMemcpyHostToDevice))) goto fail;
        if (units == 64 && Hp % 32 == 0) {
            // 32-unit interleave: a row permutation of the 64-unit planes
            std::vector<__half> h32(Whi.size()), l32(Wlo.size());
            for (int u = 0; u < Hp; ++u)
                for (int g = 0; g < 4; ++g) {
                    const size_t n64 = (size_t)(u / 64) * 256 + (size_t)g * 64 + (u % 64);
                    const size_t n32 = (size_t)(u / 32) * 128 + (size_t)g * 32 + (u % 32);
                    std::memcpy(&h32[n32 * K], &Whi[n64 * K], (size_t)K * 2);
                    std::memcpy(&l32[n32 * K], &Wlo[n64 * K], (size_t)K * 2);
                }
            if ((e = out.Whi32.ensure(h32.size() * 2)) != cudaSuccess) goto fail;
            if ((e = out.Wlo32.ensure(l32.size() * 2)) != cudaSuccess) goto fail;
            if ((e = cudaMemcpy(out.Whi32.p, h32.data(), h32.size() * 2, cudaMemcpyHostToDevice))) goto fail;
            if ((e = cudaMemcpy(out.Wlo32.p, l32.data(), l32.size() * 2, cudaMemcpyHostToDevice))) goto fail;
        }
    }
    if ((e = out.G.ensure(G.size() * 4)) != cudaSuccess) goto fail;
    if ((e = cudaMemcpy(out.G.p, G.data(), G.size() * 4, cudaMemcpyHostToDevice))) goto fail;
    return KS_OK;
fail:
    return set_error(KS_ERR_CUDA, std::string("weight upload: ") + cudaGetErrorString(e));
}

ks_status upload(DevMem& m, const void* src, size_t bytes) {
    if (m.ensure(bytes ? bytes : 4) != cudaSuccess) return set_error(KS_ERR_CUDA, "cudaMalloc failed");
    if (bytes && cudaMemcpy(m.p, src, bytes, cudaMemcpyHostToDevice) != cudaSuccess)
        return set_error(KS_ERR_CUDA, "cudaMemcpy failed");
    return KS_OK;
}

ks_status plan_enc_prefix(ks_engine& E);
}  // namespace

extern "C" ks_status ks_engine_create(const ks_model_desc* d, int32_t device, int32_t precision,
                                      ks_engine** out) {
    if (!d || !out) return set_error(KS_ERR_PARAMETER, "null argument");
    if (precision < 0 || precision > 2) return set_error(KS_ERR_PARAMETER, "unknown precision mode");
    if (d->variant != KS_VARIANT_ATTN && d->variant != KS_VARIANT_ATTN2 &&
        d->variant != KS_VARIANT_ENC_DEC && d->variant != KS_VARIANT_HYBRID2 && d->variant != KS_VARIANT_HYBRID)
        return set_error(KS_ERR_UNSUPPORTED, "unknown model variant");
    if (d->num_positions < 1 || d->num_positions > kMaxT)
        return set_error(KS_ERR_UNSUPPORTED, "number of output positions must be in [1, 16]");
    if (d->attention_dense_nodes < 1 || d->attention_dense_nodes > kMaxNd)
        return set_error(KS_ERR_UNSUPPORTED, "attention_dense_nodes must be in [1, 8]");
    if (cudaSetDevice(device) != cudaSuccess) return set_error(KS_ERR_CUDA, "cudaSetDevice failed");
    auto eng = std::make_unique<ks_engine>();
    ks_engine& E = *eng;
    E.device = device;
    E.precision = precision;
    E.variant = d->variant;
    E.n_a = d->pre_attention_size;
    E.n_s = d->post_attention_size;
    E.n_d = d->attention_dense_nodes;
    E.e = d->encoder_state_size;
    E.NA = round_up(E.n_a, 64);
    E.NS = round_up(E.n_s, 64);
    E.NE = round_up(E.e, 64);
    if (const char* u = std::getenv("KS_TC_UNITS")) E.tc_units = std::atoi(u) == 64 ? 64 : 32;
    E.T = d->num_positions;
    E.in_sizes.assign(d->input_sizes, d->input_sizes + 7);
    E.in_offset.resize(7);
    int w = 0, nin = 0;
    for (int f = 0; f < 7; ++f) {
        if (E.in_sizes[f] < 1) return set_error(KS_ERR_CHECKPOINT, "empty input vocabulary");
        E.in_offset[f] = w;
        w += E.in_sizes[f];
    }
    nin = w;
    E.d_in = w;
    E.in_values.assign(d->input_values, d->input_values + nin);
    E.vsize.assign(d->vocab_sizes, d->vocab_sizes + E.T);
    int nout = 0, fb = 1, bits_total = 0;
    E.meta.T = E.T;
    for (int p = 0; p < E.T; ++p) {
        const int V = E.vsize[p];
        if (V < 1 || V > kMaxV)
            return set_error(KS_ERR_UNSUPPORTED, "output vocabularies must have 1..32 values");
        E.meta.vsize[p] = V;
        E.meta.value_offset[p] = nout;
        E.meta.fb_offset[p] = fb;
        int b = 1;
        while ((1 << b) < V) ++b;
        E.meta.bits[p] = b;
        bits_total += b;
        nout += V;
        fb += V;
    }
    if (bits_total > 64) return set_error(KS_ERR_UNSUPPORTED, "packed prefix key exceeds 64 bits");
    int sh = 0;
    for (int p = E.T - 1; p >= 0; --p) {
        E.meta.shift[p] = sh;
        sh += E.meta.bits[p];
    }
    E.d_fb = fb;
    E.out_values.assign(d->output_values, d->output_values + nout);

    HostTensors ht;
    for (int i = 0; i < d->num_tensors; ++i)
        ht.m[d->tensor_names[i]] = {d->tensor_data[i], d->tensor_numel[i]};
    std::string err;
    ks_status st;
    if (E.variant == KS_VARIANT_HYBRID2 || E.variant == KS_VARIANT_HYBRID) {
        // packed below
    } else if (E.variant == KS_VARIANT_ENC_DEC) {
        std::vector<int> dense, slots;
        for (int k = 0; k < E.NE; ++k) dense.push_back(k < E.e ? E.d_in + k : -1);
        for (int s = 0; s < E.d_in; ++s) slots.push_back(s);
        if ((st = pack_lstm(ht, "encoder", E.d_in + E.e, E.e, E.NE, dense, slots, E.enc[0], E.precision, E.tc_units))) return st;
        dense.clear();
        slots.clear();
        for (int k = 0; k < E.NE; ++k) dense.push_back(k < E.e ? E.d_fb + k : -1);
        for (int s = 0; s < E.d_fb; ++s) slots.push_back(s);
        if ((st = pack_lstm(ht, "decoder", E.d_fb + E.e, E.e, E.NE, dense, slots, E.dec, E.precision, E.tc_units))) return st;
    } else {
        std::vector<int> dense, slots;
        for (int k = 0; k < E.NA; ++k) dense.push_back(k < E.n_a ? E.d_in + k : -1);
        for (int s = 0; s < E.d_in; ++s) slots.push_back(s);
        if ((st = pack_lstm(ht, "pre.fwd", E.d_in + E.n_a, E.n_a, E.NA, dense, slots, E.enc[0], E.precision, E.tc_units))) return st;
        if ((st = pack_lstm(ht, "pre.bwd", E.d_in + E.n_a, E.n_a, E.NA, dense, slots, E.enc[1], E.precision, E.tc_units))) return st;
        // decoder rows: [ctx (2 n_a) | fb one-hot (d_fb, attn only) | h (n_s)]  (models.cpp:215-219)
        const bool fbk = E.variant == KS_VARIANT_ATTN;
        const int hbase = 2 * E.n_a + (fbk ? E.d_fb : 0);
        const int rows = hbase + E.n_s;
        dense.clear();
        slots.clear();
        for (int k = 0; k < 2 * E.NA; ++k) {
            const int half = k / E.NA, i = k % E.NA;
            dense.push_back(i < E.n_a ? half * E.n_a + i : -1);
        }
        for (int k = 0; k < E.NS; ++k) dense.push_back(k < E.n_s ? hbase + k : -1);
        if (fbk)
            for (int s = 0; s < E.d_fb; ++s) slots.push_back(2 * E.n_a + s);
        else
            slots.push_back(-1);
        if ((st = pack_lstm(ht, "post", rows, E.n_s, E.NS, dense, slots, E.dec, E.precision, E.tc_units))) return st;
        // attention energy network: attn.hidden (n_s + 2 n_a) x n_d, attn.out n_d x 1
        const float* Wh = ht.get("attn.hidden.weights", (E.n_s + 2 * E.n_a) * E.n_d, err);
        const float* bh = ht.get("attn.hidden.bias", E.n_d, err);
        const float* wo = ht.get("attn.out.weights", E.n_d, err);
        const float* bo = ht.get("attn.out.bias", 1, err);
        if (!Wh || !bh || !wo || !bo) return set_error(KS_ERR_STATE, err);
        std::vector<float> Ws((size_t)E.NS * E.n_d, 0.0f), Wa((size_t)2 * E.NA * E.n_d, 0.0f);
        for (int i = 0; i < E.n_s; ++i)
            for (int dd = 0; dd < E.n_d; ++dd) Ws[(size_t)i * E.n_d + dd] = Wh[(size_t)i * E.n_d + dd];
        for (int k = 0; k < 2 * E.NA; ++k) {
            const int half = k / E.NA, i = k % E.NA;
            if (i >= E.n_a) continue;
            const int r = E.n_s + half * E.n_a + i;
            for (int dd = 0; dd < E.n_d; ++dd) Wa[(size_t)k * E.n_d + dd] = Wh[(size_t)r * E.n_d + dd];
        }
        if ((st = upload(E.attWs, Ws.data(), Ws.size() * 4))) return st;
        if ((st = upload(E.attWa, Wa.data(), Wa.size() * 4))) return st;
        if ((st = upload(E.attBh, bh, (size_t)E.n_d * 4))) return st;
        if ((st = upload(E.attWo, wo, (size_t)E.n_d * 4))) return st;
        E.attBo = bo[0];
    }
    if (E.variant == KS_VARIANT_HYBRID2 || E.variant == KS_VARIANT_HYBRID) {
        // conv stack over the (d_in x 7) one-hot matrix, then two bi-LSTMs (hybrid-2:
        // the second seeded with the first's final states; hybrid: over its sequence)
        E.layered = E.variant == KS_VARIANT_HYBRID;
        if (d->num_conv_layers < 1 || d->num_conv_layers > 8 || !d->conv_layers)
            return set_error(KS_ERR_UNSUPPORTED, "hybrid variants need 1..8 conv layers");
        int ch = E.d_in, len = 7, scratch = 0;
        for (int i = 0; i < d->num_conv_layers; ++i) {
            const int f = d->conv_layers[3 * i], kk = d->conv_layers[3 * i + 1], sd = d->conv_layers[3 * i + 2];
            if (f < 1 || kk < 1 || sd < 1 || len < kk)
                return set_error(KS_ERR_SHAPE, "conv stack input length shorter than kernel size");
            const int o = (len - kk) / sd + 1;
            const float* W = ht.get("conv." + std::to_string(i) + ".filters", f * ch * kk, err);
            const float* B = ht.get("conv." + std::to_string(i) + ".bias", f, err);
            if (!W || !B) return set_error(KS_ERR_STATE, err);
            E.conv_f.push_back(f);
            E.conv_k.push_back(kk);
            E.conv_s.push_back(sd);
            E.convW.emplace_back(new DevMem());
            E.convB.emplace_back(new DevMem());
            if ((st = upload(*E.convW.back(), W, (size_t)f * ch * kk * 4))) return st;
            if ((st = upload(*E.convB.back(), B, (size_t)f * 4))) return st;
            scratch = std::max(scratch, f * o);
            ch = f;
            len = o;
        }
        E.F = ch * len;
        E.FP = round_up(E.F, 64);
        E.cell = d->decoder_cell_size;
        E.CP = round_up(E.cell, 64);
        E.conv_scratch = (scratch + 3) / 4 * 4;
        std::vector<int> dense, slots{-1};
        for (int kx = 0; kx < E.FP; ++kx) dense.push_back(kx < E.F ? kx : -1);
        for (int kh = 0; kh < E.CP; ++kh) dense.push_back(kh < E.cell ? E.F + kh : -1);
        static const char* names[4] = {"bilstm1.fwd", "bilstm1.bwd", "bilstm2.fwd", "bilstm2.bwd"};
        DevLstm* dst[4] = {&E.hb1[0], &E.hb1[1], &E.hb2[0], &E.hb2[1]};
        // layered bi-LSTM 2 input = [fwd h1_t | bwd h1_t] (2 cell rows), device K layout
        // [fwd (CP) | bwd (CP) | h (CP)]
        std::vector<int> dense2;
        for (int k2 = 0; k2 < 3 * E.CP; ++k2) {
            const int part = k2 / E.CP, i = k2 % E.CP;
            dense2.push_back(i < E.cell ? part * E.cell + i : -1);
        }
        for (int q = 0; q < 4; ++q) {
            const bool two = E.layered && q >= 2;
            if ((st = pack_lstm(ht, names[q], two ? 3 * E.cell : E.F + E.cell, E.cell, E.CP, two ? dense2 : dense,
                                slots, *dst[q], E.precision, E.tc_units)))
                return st;
        }
    }
    const bool hyb = E.variant == KS_VARIANT_HYBRID2 || E.variant == KS_VARIANT_HYBRID;
    const int Hd = hyb ? 2 * E.cell : (E.variant == KS_VARIANT_ENC_DEC ? E.e : E.n_s);
    const int HdP = hyb ? 2 * E.CP : (E.variant == KS_VARIANT_ENC_DEC ? E.NE : E.NS);
    for (int p = 0; p < E.T; ++p) {
        const int V = E.vsize[p];
        const float* W = ht.get("head." + std::to_string(p) + ".weights", Hd * V, err);
        const float* b = ht.get("head." + std::to_string(p) + ".bias", V, err);
        if (!W || !b) return set_error(KS_ERR_STATE, err);
        std::vector<float> Wp((size_t)HdP * V, 0.0f);
        if (hyb) {  // feature = [fwd h (cell) | bwd h (cell)] laid out [fwd | pad | bwd | pad]
            for (int r = 0; r < Hd; ++r) {
                const int dr = r < E.cell ? r : E.CP + (r - E.cell);
                std::memcpy(Wp.data() + (size_t)dr * V, W + (size_t)r * V, sizeof(float) * (size_t)V);
            }
        } else {
            std::memcpy(Wp.data(), W, sizeof(float) * (size_t)Hd * V);
        }
        E.headW.emplace_back(new DevMem());
        E.headB.emplace_back(new DevMem());
        if ((st = upload(*E.headW.back(), Wp.data(), Wp.size() * 4))) return st;
        if ((st = upload(*E.headB.back(), b, (size_t)V * 4))) return st;
    }
    std::vector<long long> vals(E.out_values.begin(), E.out_values.end());
    if ((st = upload(E.values, vals.data(), vals.size() * 8))) return st;
    if (cudaStreamCreateWithFlags(&E.stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&E.copy_stream, cudaStreamNonBlocking) != cudaSuccess)
        return set_error(KS_ERR_CUDA, "stream creation failed");
    for (auto& b : E.io)
        if (cudaEventCreateWithFlags(&b.dec_done, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&b.copy_done, cudaEventDisableTiming) != cudaSuccess)
            return set_error(KS_ERR_CUDA, "event creation failed");
    E.beam_smem_max = 227 * 1024;
    {
        const char* cp = std::getenv("KS_CTXPROJ");
        E.ctxproj = (E.variant == KS_VARIANT_ATTN || E.variant == KS_VARIANT_ATTN2) &&
                    E.precision != KS_PREC_FP32 && !(cp && cp[0] == '0');
        E.ctxproj_force = cp && std::string(cp) == "force";
        const char* tp = std::getenv("KS_TC_PAIR");
        E.pair = tp && tp[0] == '1' && E.tc_units == 64;
        const char* kg = std::getenv("KS_GRAPHS");
        E.use_graphs = !(kg && kg[0] == '0');
        const char* pr = std::getenv("KS_TC_PAIR_AUTO");
        E.pair_auto = !(pr && pr[0] == '0');
        const char* kdp = std::getenv("KS_DEBUG_PARENTS");
        E.debug_parents = kdp && kdp[0] == '1';
        if (E.debug_parents) E.use_graphs = false;
        const char* kcp = std::getenv("KS_COMPACT");
        E.compact = !(kcp && kcp[0] == '0');
        const char* kc1 = std::getenv("KS_COMPACT_POS1");
        E.compact_pos1 = kc1 && kc1[0] == '1';
        const char* kc = std::getenv("KS_CHUNK");
        if (kc && std::atoll(kc) > 0) E.chunk = std::atoll(kc);
    }
    cudaDeviceGetAttribute(&E.num_sms, cudaDevAttrMultiProcessorCount, device);
    if (ks_status st = plan_enc_prefix(E)) return st;
    *out = eng.release();
    return KS_OK;
}

extern "C" ks_status ks_engine_create_from_checkpoint(const char* path, int32_t device,
                                                      int32_t precision, ks_engine** out) {
    ks_checkpoint* ck = nullptr;
    ks_status st = ks_checkpoint_load(path, &ck);
    if (st) return st;
    ksb_host::DescStore store;
    ks_model_desc d;
    st = ksb_host::desc_from_checkpoint(ck, store, d);
    if (!st) st = ks_engine_create(&d, device, precision, out);
    ks_checkpoint_free(ck);
    return st;
}

extern "C" void ks_engine_destroy(ks_engine* eng) {
    if (!eng) return;
    cudaSetDevice(eng->device);
    for (auto& ev : eng->prof_ev) {
        cudaEventDestroy(ev.first);
        cudaEventDestroy(ev.second);
    }
    if (eng->stream) {
        cudaStreamSynchronize(eng->stream);  // device-API decodes may still be running
        cudaStreamDestroy(eng->stream);
    }
    delete eng;
}

extern "C" int32_t ks_engine_num_positions(const ks_engine* eng) { return eng ? eng->T : 0; }
extern "C" int32_t ks_engine_vocab_size(const ks_engine* eng, int32_t p) {
    return (eng && p >= 0 && p < eng->T) ? eng->vsize[(size_t)p] : 0;
}
extern "C" int32_t ks_engine_precision(const ks_engine* eng) { return eng ? eng->precision : -1; }
extern "C" int64_t ks_engine_last_launch_count(const ks_engine* eng) { return eng ? eng->launches : 0; }
extern "C" ks_status ks_engine_set_chunk(ks_engine* eng, int64_t c) {
    if (!eng) return set_error(KS_ERR_PARAMETER, "null engine");
    std::lock_guard<std::mutex> lock(eng->mu);
    if (!eng) return set_error(KS_ERR_PARAMETER, "null engine");
    eng->chunk = c > 0 ? c : 65536;
    return KS_OK;
}

extern "C" ks_status ks_engine_synthetic_descriptors(const ks_engine* eng, uint64_t seed, int64_t start,
                                                     int64_t count, int64_t* out_desc) {
    if (!eng) return set_error(KS_ERR_PARAMETER, "null engine");
    return ks_synthetic_descriptors(eng->in_sizes.data(), eng->in_values.data(), seed, start, count, out_desc);
}

extern "C" ks_status ks_encode_problems(const ks_engine* eng, const int64_t* desc, int64_t B,
                                        int32_t allow_nearest, int32_t* tok, int64_t* bad_row) {
    static const char* names[7] = {"n", "c", "h", "w", "k", "y", "x"};
    if (!eng || (!desc && B) || (!tok && B)) return set_error(KS_ERR_PARAMETER, "null argument");
    for (int64_t b = 0; b < B; ++b) {
        for (int f = 0; f < 7; ++f) {
            const int64_t v = desc[b * 7 + f];
            if (v < 1) {
                if (bad_row) *bad_row = b;
                return set_error(KS_ERR_VALIDATION,
                                 std::string("descriptor field ") + names[f] + " must be >= 1, got " +
                                     std::to_string(v),
                                 names[f]);
            }
            const int64_t* vals = eng->in_values.data() + eng->in_offset[(size_t)f];
            const int n = eng->in_sizes[(size_t)f];
            int id = -1;
            for (int i = 0; i < n; ++i)
                if (vals[i] == v) { id = i; break; }
            // FieldVocab::nearest (encoding.cpp:26-34): closest, smaller value on ties
            int64_t best = vals[0];
            for (int i = 0; i < n; ++i) {
                const int64_t dv = vals[i] > v ? vals[i] - v : v - vals[i];
                const int64_t db = best > v ? best - v : v - best;
                if (dv < db || (dv == db && vals[i] < best)) best = vals[i];
            }
            if (id < 0 && allow_nearest)
                for (int i = 0; i < n; ++i)
                    if (vals[i] == best) { id = i; break; }
            if (id < 0) {
                if (bad_row) *bad_row = b;
                return set_error(KS_ERR_VALIDATION,
                                 "value " + std::to_string(v) + " of field " + names[f] +
                                     " is not in the vocabulary (nearest known: " +
                                     std::to_string(best) + ")",
                                 names[f]);
            }
            tok[b * 7 + f] = id;
        }
    }
    return KS_OK;
}

// ---------------------------------------------------------------------------
// decode schedule
// ---------------------------------------------------------------------------
namespace {

struct PredDev {
    int n = 0;
    int n_terms = 0;
    int n_bytes = 0;
    bool needs_desc = false;
    bool has_host = false;
    ks_host_pred_fn hook = nullptr;
    void* user = nullptr;
};

ks_status upload_preds(ks_engine& E, const ks_pred* preds, int n, PredDev& pd) {
    std::vector<DevPred> dp;
    std::vector<unsigned char> bytes;
    std::vector<int> tpos, tfield;
    std::vector<double> tw;
    int total_v = 0;
    for (int p = 0; p < E.T; ++p) total_v += E.vsize[(size_t)p];
    for (int i = 0; i < n; ++i) {
        const ks_pred& q = preds[i];
        DevPred d{};
        d.kind = q.kind;
        d.full = q.full_sequence_only ? 1 : 0;
        if (q.kind == KS_PRED_MASK) {
            if (!q.allowed) return set_error(KS_ERR_PARAMETER, "mask predicate without table");
            d.allowed_off = (int)bytes.size();
            bytes.insert(bytes.end(), q.allowed, q.allowed + total_v);
        } else if (q.kind == KS_PRED_BUDGET || q.kind == KS_PRED_PRODUCT || q.kind == KS_PRED_DIVIDES) {
            if (q.n_terms < 0 || (q.n_terms > 0 && !q.term_pos))
                return set_error(KS_ERR_PARAMETER, "predicate terms missing");
            d.n_terms = q.n_terms;
            d.terms_off = (int)tpos.size();
            for (int t = 0; t < q.n_terms; ++t) {
                const int pp = q.term_pos[t];
                if (pp < -1 || pp >= E.T) return set_error(KS_ERR_INDEX, "predicate term position out of range");
                tpos.push_back(pp);
                tw.push_back(q.kind == KS_PRED_BUDGET ? (q.term_w ? q.term_w[t] : 0.0) : 0.0);
                int f = 0;
                if (q.kind == KS_PRED_DIVIDES) {
                    if (!q.term_field) return set_error(KS_ERR_PARAMETER, "divisibility predicate without fields");
                    f = q.term_field[t];
                    if (f < 0 || f > 6) return set_error(KS_ERR_INDEX, "descriptor field out of range");
                    pd.needs_desc = true;
                }
                tfield.push_back(f);
            }
            if (q.kind == KS_PRED_BUDGET) {
                for (int t = 0; t < q.n_terms; ++t)
                    if (q.term_w && q.term_w[t] < 0.0)
                        return set_error(KS_ERR_PARAMETER, "resource budget weight must be nonnegative");
                if (q.budget < 0.0) return set_error(KS_ERR_PARAMETER, "resource budget must be nonnegative");
            }
            d.budget = q.budget;
            d.scale = q.scale;
            d.limit = q.limit;
        } else if (q.kind == KS_PRED_HOST) {
            pd.has_host = true;
        } else {
            return set_error(KS_ERR_PARAMETER, "unknown predicate kind " + std::to_string(q.kind));
        }
        dp.push_back(d);
    }
    pd.n = n;
    pd.n_terms = (int)tpos.size();
    pd.n_bytes = (int)bytes.size();
    std::vector<unsigned char> blob;
    auto put = [&](const void* p, size_t nb) {
        const size_t o = blob.size();
        blob.resize(o + nb + 8);
        std::memcpy(blob.data() + o, &nb, 8);
        if (nb) std::memcpy(blob.data() + o + 8, p, nb);
    };
    put(dp.data(), dp.size() * sizeof(DevPred));
    put(bytes.data(), bytes.size());
    put(tpos.data(), tpos.size() * 4);
    put(tw.data(), tw.size() * 8);
    put(tfield.data(), tfield.size() * 4);
    if (blob == E.pred_blob && E.preds.p) return KS_OK;  // tables already on the device
    // the engine stream may still be reading the previous tables (device API calls
    // return before their kernels finish)
    KS_CUDA(cudaStreamSynchronize(E.stream));
    E.pred_blob.clear();
    ks_status st;
    if ((st = upload(E.preds, dp.data(), dp.size() * sizeof(DevPred)))) return st;
    if ((st = upload(E.pbytes, bytes.data(), bytes.size()))) return st;
    if ((st = upload(E.tpos, tpos.data(), tpos.size() * 4))) return st;
    if ((st = upload(E.tw, tw.data(), tw.size() * 8))) return st;
    if ((st = upload(E.tfield, tfield.data(), tfield.size() * 4))) return st;
    E.pred_blob = std::move(blob);
    return KS_OK;
}

// shared-prefix encoder tables of a C-config chunk: covered[d] = the last step of
// direction d that runs per prefix (steps with no more prefixes than configs), byte
// offsets of h fp32 / hi / lo [sum R][He], the c ping-pong [2][maxr][He] fp32 and
// the replicated parent planes [2][maxr][He] fp16
size_t prefix_layout(const ks_engine& E, int64_t C, int covered[2], size_t at[2][5], size_t maxr[2]) {
    const int He = E.NA;
    size_t bytes = 0;
    for (int d = 0; d < 2; ++d) {
        const ks_engine::EncTable& T = E.etab[d];
        int S = -1;
        while (C >= E.prefix_min && S < T.S && T.R[S + 1] <= C) ++S;
        covered[d] = S;
        maxr[d] = 0;
        for (int i = 0; i < 5; ++i) at[d][i] = bytes;
        if (S < 0) continue;
        const size_t rows = (size_t)(T.off[S] + T.R[S]);
        for (int j = 0; j <= S; ++j) maxr[d] = std::max(maxr[d], (size_t)T.R[j]);
        at[d][1] = at[d][0] + rows * He * 4;
        at[d][2] = at[d][1] + rows * He * 2;
        at[d][3] = at[d][2] + rows * He * 2;
        at[d][4] = at[d][3] + 2 * maxr[d] * He * 4;  // replicated parent planes [2][maxr][He]
        bytes = at[d][4] + 2 * maxr[d] * He * 2;
    }
    return bytes;
}

ks_status ensure_workspace(ks_engine& E, int64_t C, int k) {
    const int64_t R = C * k;
    const bool enc_dec = E.variant == KS_VARIANT_ENC_DEC;
    const int Hd = enc_dec ? E.NE : E.NS;
    const int NA2 = enc_dec ? 0 : 2 * E.NA;
    const int Kd = NA2 + Hd;
    const int He = enc_dec ? E.NE : E.NA;
    cudaError_t e = cudaSuccess;
#define ENS(buf, n) do { if ((e = (buf).ensure((size_t)(n))) != cudaSuccess) goto fail; } while (0)
    ENS(E.tok, C * 7 * 4);
    ENS(E.desc, C * 7 * 8);
    if (E.variant == KS_VARIANT_HYBRID2 || E.variant == KS_VARIANT_HYBRID) {
        const int64_t K = E.FP + E.CP;
        if (E.layered) {
            const int64_t K2 = 3LL * E.CP;
            ENS(E.hybH1, (int64_t)E.T * C * 2 * E.CP * 4);
            ENS(E.hybX2, E.precision == KS_PREC_FP32 ? 2LL * E.T * C * K2 * 4 : 2LL * 2 * E.T * C * K2 * 2);
        }
        if (E.precision == KS_PREC_FP32) {
            ENS(E.hybAf, 4 * C * K * 4);            // [dir*2 + pingpong][C][K] fp32
        } else {
            ENS(E.hybA, 2 * 4 * C * K * 2);         // [hi/lo][dir*2 + pingpong][C][K] fp16
        }
        ENS(E.hybC, 4 * C * E.CP * 4);              // [dir][pingpong][C][CP]
        ENS(E.hybH, 2 * C * E.CP * 4);              // bi-LSTM 1 h scratch [dir][C][CP]
        ENS(E.feat, (int64_t)E.T * C * 2 * E.CP * 4);  // [T][C][fwd | bwd]
    } else {
        ENS(E.act, C * 7 * (enc_dec ? E.NE : NA2) * 4);
        ENS(E.uatt, C * 7 * E.n_d * 4 + 16);
        ENS(E.encc, 2 * 2 * C * He * 4);
        if (E.etab[0].S >= 0 || E.etab[1].S >= 0) {
            int cov[2];
            size_t at[2][5], maxr[2];
            ENS(E.encp, prefix_layout(E, C, cov, at, maxr));
        }
        ENS(E.encA, 2 * 2 * 2 * C * He * 2);   // [dir][pingpong][hi/lo][C][He] fp16
        if (E.precision == KS_PREC_FP32) {
            ENS(E.Abuf, R * Kd * 4);
        } else {
            const int64_t lda = E.ctxproj ? std::max<int64_t>(Kd, E.alpha_cols_of(1) + Hd) : Kd;
            ENS(E.Ahi, R * lda * 2);
            ENS(E.Alo, R * lda * 2);
        }
        ENS(E.hbuf, 2 * R * Hd * 4);
        ENS(E.cbuf, 2 * R * Hd * 4);
        if (E.ctxproj) {
            ENS(E.cpbuf, (2 * C + 2 + 4 * R) * 4 + R * 16 + 16);
            const int64_t ldt = (C * 7 + 7) / 8 * 8;
            ENS(E.Pt, 2 * 4 * (int64_t)Hd * ldt * 2);   // [hi/lo][4NS][ldt] fp16
            ENS(E.actA, 2 * C * 7 * (int64_t)NA2 * 2);
        }
    }
    for (int i = 0; i < 2; ++i) {
        ENS(E.live[i], R);
        ENS(E.lp[i], R * 8);
        ENS(E.key[i], R * 8);
        ENS(E.parent[i], R * 4);
        ENS(E.slot[i], R * 4);
    }
    ENS(E.status, C * 4);
    ENS(E.fpred, C * 4);
    ENS(E.fstep, C * 4);
#undef ENS
    return KS_OK;
fail:
    return set_error(KS_ERR_CUDA, std::string("workspace allocation: ") + cudaGetErrorString(e));
}

ks_status launch_lstm(ks_engine& E, const LstmArgs& a0, const LstmArgs* a1, DevLstm& L0,
                      DevLstm* L1, double useful_flops) {
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    const bool timed = E.prof && a0.K > 0;
    if (timed) {
        cudaEventCreate(&ev0);
        cudaEventCreate(&ev1);
        cudaEventRecord(ev0, E.stream);
    }
    int n = 0;
    bool done = false;
    if (E.precision != KS_PREC_FP32 && a0.K > 0) {
        const bool u32 = E.units_now == 32 && E.tc_units == 64;  // 32-unit planes of 64-unit packings
        auto whi = [&](DevLstm& L) { return (u32 ? L.Whi32 : L.Whi).as<__half>(); };
        auto wlo = [&](DevLstm& L) { return (u32 ? L.Wlo32 : L.Wlo).as<__half>(); };
        done = launch_lstm_tc(a0, a1, E.precision, whi(L0), wlo(L0), L1 ? whi(*L1) : nullptr,
                              L1 ? wlo(*L1) : nullptr, E.stream, &n, E.units_now,
                              E.pair_now() || (E.pair_auto && E.units_now == 64 && a0.kb_alpha == 0 &&
                                               a0.fan <= 1 && !a0.cp_M && (!a1 || (a1->kb_alpha == 0 && a1->fan <= 1))));
        if (!done) return set_error(KS_ERR_CUDA, "tensor-core GEMM launch failed");
    }
    if (!done && a0.K == 0 && launch_lstm_k0(a0, a1, E.num_sms, E.stream)) {
        done = true;
        n = 1;
    }
    if (!done) {
        dim3 grid((unsigned)((a0.M + SB_M_HOST - 1) / SB_M_HOST), (unsigned)(a0.H / 32), a1 ? 2u : 1u);
        lstm_step_simt<<<grid, 256, 0, E.stream>>>(a0, a1 ? *a1 : a0);
        n = 1;
    }
    E.launches += n;
    if (timed) {
        cudaEventRecord(ev1, E.stream);
        E.prof_ev.emplace_back(ev0, ev1);
        E.prof_flops.push_back(useful_flops);
        // FLOPs the tensor pipe issues: 2 M K 4H per MMA pass (3 passes in F16X3); in
        // alpha-block mode K varies per 128-row tile (tile_k, ks_gemm_tc.cu)
        auto exec_of = [&](const LstmArgs& a) {
            if (a.K <= 0) return 0.0;
            const double passes = E.precision == KS_PREC_F16X3 ? 3.0 : 1.0;
            double rowk = (double)a.M * a.K;
            if (a.cp_M) {
                // compacted rows: the row count and the tiles' configs are device data
                // (profiling runs only: a synchronous read-back)
                int mc = 0;
                cudaMemcpyAsync(&mc, a.cp_M, 4, cudaMemcpyDeviceToHost, E.stream);
                cudaStreamSynchronize(E.stream);
                std::vector<int> cfg((size_t)std::max(mc, 1));
                cudaMemcpy(cfg.data(), a.cp_cfg, (size_t)mc * 4, cudaMemcpyDeviceToHost);
                rowk = 0.0;
                for (int r0 = 0; r0 < mc; r0 += a.alpha_tile) {
                    const int r1 = std::min(mc, r0 + a.alpha_tile);
                    const int x0 = (7 * cfg[(size_t)r0]) & ~7;
                    const int kba = std::min(a.kb_alpha, (7 * (cfg[(size_t)r1 - 1] + 1) - x0 + kTcBK - 1) / kTcBK);
                    rowk += (double)(r1 - r0) * (a.K - (double)kTcBK * (a.kb_alpha - kba));
                }
                return 2.0 * rowk * 4.0 * a.H * passes;
            }
            if (a.kb_alpha > 0) {
                rowk = 0.0;
                const int TR = a.alpha_tile;
                for (int mt = 0; mt * TR < a.M; ++mt) {
                    const int b0 = mt * TR / a.rows_per_cfg, b1 = (mt * TR + TR - 1) / a.rows_per_cfg;
                    const int x0 = (7 * b0) & ~7;
                    const int kba = std::min(a.kb_alpha, (7 * (b1 + 1) - x0 + kTcBK - 1) / kTcBK);
                    const int rows = std::min(TR, a.M - mt * TR);
                    rowk += (double)rows * (a.K - (double)kTcBK * (a.kb_alpha - kba));
                }
            }
            return 2.0 * rowk * 4.0 * a.H * passes;
        };
        E.prof_exec.push_back(exec_of(a0) + (a1 ? exec_of(*a1) : 0.0));
    }
    const cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return set_error(KS_ERR_CUDA, std::string("lstm launch: ") + cudaGetErrorString(err));
    return KS_OK;
}

// hybrid encoders: conv stack, bi-LSTM 1 over T_out copies of the encoding;
// hybrid-2: bi-LSTM 2 over the same copies seeded with bi-LSTM 1's final
// states (models.cpp:296-371, 422-425); hybrid: bi-LSTM 2 over bi-LSTM 1's
// activation sequence from a zero state (models.cpp:409-418).  Writes the
// per-position features [fwd h_t | bwd h_t].
ks_status encode_hybrid(ks_engine& E, int64_t C, const int* d_tok) {
    cudaStream_t s = E.stream;
    const int T = E.T, CP = E.CP, FP = E.FP;
    const int64_t K = FP + CP;
    const bool split = E.precision != KS_PREC_FP32;
    __half* hybA = E.hybA.as<__half>();
    auto Ahi = [&](int dir, int pp) { return hybA + ((size_t)(dir * 2 + pp)) * C * K; };
    auto Alo = [&](int dir, int pp) { return hybA + ((size_t)(4 + dir * 2 + pp)) * C * K; };
    auto Af = [&](int dir, int pp) { return E.hybAf.as<float>() + ((size_t)(dir * 2 + pp)) * C * K; };
    auto Cb = [&](int dir, int pp) { return E.hybC.as<float>() + ((size_t)(dir * 2 + pp)) * C * CP; };
    ConvArgs ca{};
    ca.C = (int)C;
    ca.n_conv = (int)E.conv_f.size();
    for (int i = 0; i < ca.n_conv; ++i) {
        ca.f[i] = E.conv_f[(size_t)i];
        ca.k[i] = E.conv_k[(size_t)i];
        ca.s[i] = E.conv_s[(size_t)i];
        ca.W[i] = E.convW[(size_t)i]->as<float>();
        ca.b[i] = E.convB[(size_t)i]->as<float>();
    }
    ca.d_in = E.d_in;
    for (int f = 0; f < 7; ++f) ca.in_offset[f] = E.in_offset[(size_t)f];
    ca.tok = d_tok;
    ca.F = E.F;
    ca.FP = FP;
    ca.CP = CP;
    ca.K = (int)K;
    ca.split_mode = E.precision == KS_PREC_FP32 ? 0 : (E.precision == KS_PREC_F16X3 ? 1 : 2);
    for (int q = 0; q < 4; ++q) {
        ca.Ahi[q] = split ? Ahi(q / 2, q % 2) : nullptr;
        ca.Alo[q] = split ? Alo(q / 2, q % 2) : nullptr;
        ca.Af[q] = split ? nullptr : Af(q / 2, q % 2);
    }
    ca.scratch_floats = E.conv_scratch;
    if (!launch_hybrid_conv(ca, s)) return set_error(KS_ERR_UNSUPPORTED, "conv stack too large for the conv kernel");
    E.launches++;
    ks_status st;
    // layered (hybrid): bi-LSTM 2 operands [fwd h1_t | bwd h1_t | h2] per direction and step
    const int64_t K2 = 3LL * CP;
    auto X2hi = [&](int dir, int t) { return E.hybX2.as<__half>() + ((size_t)(dir * T + t)) * C * K2; };
    auto X2lo = [&](int dir, int t) { return E.hybX2.as<__half>() + ((size_t)((2 + dir) * T + t)) * C * K2; };
    auto X2f = [&](int dir, int t) { return E.hybX2.as<float>() + ((size_t)(dir * T + t)) * C * K2; };
    float* H1 = E.layered ? E.hybH1.as<float>() : nullptr;
    for (int step = 0; step < 2 * T; ++step) {
        const bool second = step >= T;
        const int cur = step & 1, nxt = cur ^ 1;
        if (E.layered && step == T) {
            HybPackArgs hp{};
            hp.H1 = H1;
            hp.C = (int)C;
            hp.T = T;
            hp.CP = CP;
            hp.split_mode = ca.split_mode;
            for (int dir = 0; dir < 2; ++dir) {
                hp.Xhi[dir] = split ? X2hi(dir, 0) : nullptr;
                hp.Xlo[dir] = split ? X2lo(dir, 0) : nullptr;
                hp.Xf[dir] = split ? nullptr : X2f(dir, 0);
            }
            if (!launch_hybrid_pack(hp, s)) return set_error(KS_ERR_CUDA, "hybrid pack launch failed");
            E.launches++;
        }
        LstmArgs a[2];
        for (int dir = 0; dir < 2; ++dir) {
            LstmArgs& p = a[dir];
            std::memset(&p, 0, sizeof p);
            p.M = (int)C;
            p.H = CP;
            p.K = (int)K;
            p.A = split ? nullptr : Af(dir, cur);
            p.lda = K;
            p.A_hi = split ? Ahi(dir, cur) : nullptr;
            p.A_lo = split ? Alo(dir, cur) : nullptr;
            const int t = second ? (dir == 0 ? step - T : T - 1 - (step - T)) : (dir == 0 ? step : T - 1 - step);
            if (E.layered && second) {
                p.K = (int)K2;
                p.lda = K2;
                p.A = split ? nullptr : X2f(dir, t);
                p.A_hi = split ? X2hi(dir, t) : nullptr;
                p.A_lo = split ? X2lo(dir, t) : nullptr;
            }
            DevLstm& L = second ? E.hb2[dir] : E.hb1[dir];
            p.W = L.W.as<float>();
            p.G = L.G.as<float>();
            p.slot_ptr = nullptr;
            p.slot_base = 0;
            p.c_prev = (step == 0 || (E.layered && step == T)) ? nullptr : Cb(dir, nxt);
            p.ldc_prev = CP;
            p.c_out = Cb(dir, cur);
            p.ldc = CP;
            // the new h feeds the next step's operand (h part of the other buffer)
            if (split) {
                p.hA_hi = Ahi(dir, nxt) + FP;
                p.hA_lo = Alo(dir, nxt) + FP;
                p.ldha = K;
                p.ha_bf16 = E.precision == KS_PREC_BF16 ? 1 : 0;
            }
            float* next_f32 = split ? nullptr : Af(dir, nxt) + FP;
            if (E.layered && second) {
                // the next step of this direction reads h from its own operand buffer
                const int tn = dir == 0 ? t + 1 : t - 1;
                const bool more = tn >= 0 && tn < T;
                p.hA_hi = (split && more) ? X2hi(dir, tn) + 2 * CP : nullptr;
                p.hA_lo = (split && more) ? X2lo(dir, tn) + 2 * CP : nullptr;
                p.ldha = K2;
                next_f32 = (!split && more) ? X2f(dir, tn) + 2 * CP : nullptr;
            }
            if (!second) {
                if (E.layered) {  // bi-LSTM 1's sequence feeds bi-LSTM 2
                    p.h_out = H1 + (size_t)t * C * 2 * CP + (size_t)dir * CP;
                    p.ldh = 2 * CP;
                    p.h_out2 = next_f32;
                    p.ldh2 = K;
                } else {
                    p.h_out = split ? E.hybH.as<float>() + (size_t)dir * C * CP : next_f32;
                    p.ldh = split ? CP : K;
                }
            } else {
                p.h_out = E.feat.as<float>() + (size_t)t * C * 2 * CP + (size_t)dir * CP;
                p.ldh = 2 * CP;
                p.h_out2 = next_f32;
                p.ldh2 = E.layered ? K2 : K;
            }
        }
        if (step == 0 && !split) {
            // FP32 mode: the step-0 operand's h part is zero (written by the conv kernel)
        }
        const double fl = 2.0 * 2.0 * (double)C * ((E.layered && second) ? 3 * E.cell : E.F + E.cell) * 4.0 * E.cell;
        if ((st = launch_lstm(E, a[0], &a[1], second ? E.hb2[0] : E.hb1[0], second ? &E.hb2[1] : &E.hb1[1], fl)))
            return st;
    }
    return KS_OK;
}

// Decodes one chunk of C configs already resident on the device.
// ---- shared-prefix encoder
// Prefix r of step j (0 <= r < R_j) is numbered with the newest digit least
// significant: r = parent * size_j + digit_j, parent = the step-(j-1) prefix, so a
// config's row at step j is Horner's ((tok_0 * size_1 + tok_1) * size_2 + ...) over
// the fields it has read.  Step j is one gate-GEMM launch over its R_j prefixes:
// A row r = the split h of parent r / size_j (the parent planes replicated by
// enc_prefix_replicate), c_prev through the parent index, slot = digit_j.  (A
// fan-out epilogue over the R_{j-1} parents does fewer MMAs but its per-child loop is
// latency-bound: 2-4x slower at these sizes, tools/tiny_gemm.cu.)  The digit and
// parent arrays depend on the vocabulary sizes only; the states are computed per chunk.
ks_status plan_enc_prefix(ks_engine& E) {
    const char* env = std::getenv("KS_ENC_PREFIX");
    const bool on = E.ctxproj && E.precision != KS_PREC_FP32 && !(env && env[0] == '0');
    if (!on) return KS_OK;
    const int He = E.NA;
    if (const char* pm = std::getenv("KS_ENC_PREFIX_MIN")) E.prefix_min = std::atoll(pm);
    // prefix table elements (h fp32 + split h: 8 B each) and per-step rows x units
    const int64_t kCapStep = 1LL << 24, kCapTotal = 6LL << 24;
    for (int dir = 0; dir < 2; ++dir) {
        ks_engine::EncTable& T = E.etab[dir];
        T.S = -1;
        int64_t r = 1, total = 0;
        for (int j = 0; j < 7; ++j) {
            const int t = dir == 0 ? j : 6 - j;
            const int64_t r2 = r * E.in_sizes[(size_t)t];
            if (r2 * He > kCapStep || (total + r2) * He > kCapTotal) break;
            T.order[j] = t;
            T.size[j] = E.in_sizes[(size_t)t];
            T.R[j] = r2;
            T.off[j] = total;
            total += r2;
            r = r2;
            T.S = j;
        }
        if (T.S < 0) continue;
        T.total = total;
        std::vector<int> dg((size_t)total * 2);
        for (int j = 0; j <= T.S; ++j)
            for (int64_t x = 0; x < T.R[j]; ++x) {
                dg[(size_t)(T.off[j] + x)] = (int)(x % T.size[j]);
                dg[(size_t)(total + T.off[j] + x)] = (int)(x / T.size[j]);
            }
        if (T.digits.ensure(dg.size() * 4)) return set_error(KS_ERR_CUDA, "prefix digit allocation failed");
        KS_CUDA(cudaMemcpy(T.digits.p, dg.data(), dg.size() * 4, cudaMemcpyHostToDevice));
    }
    return KS_OK;
}

struct EncGatherArgs {
    const int* tok;              // [C][7]
    int C, He, S[2];
    int order[2][7];
    int size[2][7];
    long long off[2][7];
    const float* h[2];           // prefix tables [sum R][He] per direction
    const __half* hi[2];
    const __half* lo[2];
    const float* c[2];           // c of step S[dir] [R_S][He]
    float* act;                  // a_t fp32, row stride act_ld, step t at t*NA2 + dir*NA
    __half* ahi;                 // a_t operand planes (same layout)
    __half* alo;
    long long act_ld, NA2, NA;
    float* c_last[2];            // the encoder loop's c slot of step S[dir]
};

// one warp per (config, prefix-computed direction-step); lanes stride over 8-unit groups
__global__ void __launch_bounds__(256) enc_prefix_gather(EncGatherArgs a) {
    const int q8 = a.He / 8;
    const int steps = a.S[0] + 1 + a.S[1] + 1;
    const int lane = threadIdx.x & 31;
    const unsigned n = (unsigned)a.C * steps;
    for (unsigned w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n; w += (gridDim.x * blockDim.x) >> 5) {
        const int j = (int)(w % steps);
        const int b = (int)(w / steps);
        const int d = j <= a.S[0] ? 0 : 1;
        const int s = d == 0 ? j : j - (a.S[0] + 1);
        const int* tk = a.tok + (size_t)b * 7;
        long long row = 0;
        for (int x = 0; x <= s; ++x) row = row * a.size[d][x] + __ldg(tk + a.order[d][x]);
        const int t = a.order[d][s];
        const size_t src0 = ((size_t)a.off[d][s] + row) * a.He;
        const size_t dst0 = (size_t)b * a.act_ld + t * a.NA2 + d * a.NA;
        for (int q = lane; q < q8; q += 32) {
            const size_t src = src0 + q * 8, dst = dst0 + q * 8;
            const float4* hs = reinterpret_cast<const float4*>(a.h[d] + src);
            float4* hd = reinterpret_cast<float4*>(a.act + dst);
            hd[0] = __ldg(hs);
            hd[1] = __ldg(hs + 1);
            *reinterpret_cast<uint4*>(a.ahi + dst) = __ldg(reinterpret_cast<const uint4*>(a.hi[d] + src));
            *reinterpret_cast<uint4*>(a.alo + dst) = __ldg(reinterpret_cast<const uint4*>(a.lo[d] + src));
            if (s == a.S[d]) {
                const float4* cs = reinterpret_cast<const float4*>(a.c[d] + (size_t)row * a.He + q * 8);
                float4* cd = reinterpret_cast<float4*>(a.c_last[d] + (size_t)b * a.He + q * 8);
                cd[0] = __ldg(cs);
                cd[1] = __ldg(cs + 1);
            }
        }
    }
}

// A operand of a prefix step: row r of the step = the split h of parent r / fan
struct RepJob {
    const __half* src_hi;
    const __half* src_lo;
    __half* dst_hi;
    __half* dst_lo;
    long long rows;
    int fan;
};

__global__ void __launch_bounds__(256) enc_prefix_replicate(RepJob j0, RepJob j1, int He) {
    const RepJob& j = blockIdx.y == 0 ? j0 : j1;
    const int q8 = He / 8;
    const long long n = j.rows * q8;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / q8;
        const int q = (int)(i - r * q8);
        const size_t src = (size_t)(r / j.fan) * He + q * 8, dst = (size_t)r * He + q * 8;
        *reinterpret_cast<uint4*>(j.dst_hi + dst) = __ldg(reinterpret_cast<const uint4*>(j.src_hi + src));
        *reinterpret_cast<uint4*>(j.dst_lo + dst) = __ldg(reinterpret_cast<const uint4*>(j.src_lo + src));
    }
}

// ---- parent compaction (alpha-block positions)
// Row b*H + i of a position is child i of config b; siblings (same parent) share the
// gate GEMM's A row ([alpha | h_prev]: attention runs on the parent's h) and c_prev.
// cp_count: distinct live parents per config (>= 1: a config without live rows keeps
// one dummy row, so a 128-row GEMM tile spans at most 128 configs and the alpha block
// stays within alpha_cols_for(128, 1) columns), and each block's total.
__device__ __forceinline__ int cp_distinct(const int* pa, const unsigned char* lv, int H) {
    int n = 0;
    for (int i = 0; i < H; ++i) {
        if (!lv[i]) continue;
        bool seen = false;
        for (int j = 0; j < i && !seen; ++j) seen = lv[j] && pa[j] == pa[i];
        n += !seen;
    }
    return n > 0 ? n : 1;
}

__global__ void __launch_bounds__(256) cp_count(const int* __restrict__ parent, const unsigned char* __restrict__ live,
                                                int C, int H, int* __restrict__ cnt, int* __restrict__ part) {
    __shared__ int ws[8];
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    int n = 0;
    if (b < C) {
        n = cp_distinct(parent + (size_t)b * H, live + (size_t)b * H, H);
        cnt[b] = n;
    }
    int x = n;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < 8; ++w) t += ws[w];
        part[blockIdx.x] = t;
    }
}

// compacted rows of config b from base_b = (totals of the previous blocks) + (the
// block's exclusive scan); parents in first-occurrence order, each row's children
// {row, slot} grouped in child[b*H ..]; the last block writes the row count
__global__ void __launch_bounds__(256) cp_fill(const int* __restrict__ parent, const unsigned char* __restrict__ live,
                                               const int* __restrict__ slot, int C, int H,
                                               const int* __restrict__ cnt, const int* __restrict__ part,
                                               int* __restrict__ total, int* __restrict__ cfg,
                                               int* __restrict__ prow, int* __restrict__ cstart,
                                               int* __restrict__ ccount, int4* __restrict__ child) {
    __shared__ int ws[8];
    __shared__ int off_s;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (warp == 0) {
        int t = 0;
        for (int j = lane; j < (int)blockIdx.x; j += 32) t += part[j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) off_s = t;
    }
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    const int n = b < C ? cnt[b] : 0;
    int x = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    int pre = off_s;
    for (int w = 0; w < warp; ++w) pre += ws[w];
    int rc = pre + x - n;
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == blockDim.x - 1) *total = rc + n;
    if (b >= C) return;
    const int* pa = parent + (size_t)b * H;
    const unsigned char* lv = live + (size_t)b * H;
    int q = b * H;
    bool any = false;
    for (int i = 0; i < H; ++i) {
        if (!lv[i]) continue;
        bool seen = false;
        for (int j = 0; j < i && !seen; ++j) seen = lv[j] && pa[j] == pa[i];
        if (seen) continue;
        any = true;
        cfg[rc] = b;
        prow[rc] = pa[i];
        cstart[rc] = q;
        int m = 0;
        for (int j = i; j < H; ++j)
            if (lv[j] && pa[j] == pa[i]) {
                child[q++] = make_int4(b * H + j, slot ? slot[(size_t)b * H + j] : 0, rc, pa[i]);
                ++m;
            }
        ccount[rc] = m;
        ++rc;
    }
    if (!any) {  // the dummy row of a config without live rows
        cfg[rc] = b;
        prow[rc] = -1;
        cstart[rc] = q;
        ccount[rc] = 0;
    }
    // entries of dead children: skipped by the epilogue (it walks entry ranges)
    for (; q < (b + 1) * H; ++q) child[q] = make_int4(-1, 0, -1, -1);
}

__global__ void dbg_parents(const int* parent, const unsigned char* live, int C, int H, unsigned long long* acc) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= C) return;
    int n = 0, nl = 0;
    for (int i = 0; i < H; ++i) {
        if (!live[(size_t)b * H + i]) continue;
        ++nl;
        bool seen = false;
        for (int j = 0; j < i; ++j)
            if (live[(size_t)b * H + j] && parent[(size_t)b * H + j] == parent[(size_t)b * H + i]) seen = true;
        n += !seen;
    }
    atomicAdd(acc, (unsigned long long)n);
    atomicAdd(acc + 1, (unsigned long long)nl);
}

// Runs the prefix steps of both directions (step s of every direction that covers
// it in one launch) and gathers every config's states of those steps into a_t, its
// operand planes and the encoder loop's c slot.  covered[d] = the last such step.
ks_status encode_prefix(ks_engine& E, int64_t C, const int* d_tok, float* act, __half* ahi, __half* alo,
                        long long act_ld, int NA2, float* c_slot0, float* c_slot1, int covered[2]) {
    const int He = E.NA;
    size_t at[2][5], maxr[2];
    const size_t bytes = prefix_layout(E, C, covered, at, maxr);
    if (covered[0] < 0 && covered[1] < 0) return KS_OK;
    if (E.encp.ensure(bytes)) return set_error(KS_ERR_CUDA, "prefix table allocation failed");
    char* base = E.encp.as<char>();
    auto H = [&](int d) { return reinterpret_cast<float*>(base + at[d][0]); };
    auto HI = [&](int d) { return reinterpret_cast<__half*>(base + at[d][1]); };
    auto LO = [&](int d) { return reinterpret_cast<__half*>(base + at[d][2]); };
    auto CB = [&](int d, int s) { return reinterpret_cast<float*>(base + at[d][3]) + (size_t)(s & 1) * maxr[d] * He; };
    auto REP = [&](int d) { return reinterpret_cast<__half*>(base + at[d][4]); };
    ks_status st;
    for (int s = 0; s <= std::max(covered[0], covered[1]); ++s) {
        LstmArgs a[2];
        int na = 0, dd[2];
        RepJob rj[2];
        int nr = 0;
        for (int d = 0; d < 2; ++d) {
            if (s > covered[d]) continue;
            const ks_engine::EncTable& T = E.etab[d];
            LstmArgs& p = a[na];
            dd[na++] = d;
            std::memset(&p, 0, sizeof p);
            const size_t prev = s ? (size_t)T.off[s - 1] * He : 0, cur = (size_t)T.off[s] * He;
            const bool rep = s > 0 && T.size[s] > 1;
            if (rep) {
                RepJob& j = rj[nr++];
                j.src_hi = HI(d) + prev;
                j.src_lo = LO(d) + prev;
                j.dst_hi = REP(d);
                j.dst_lo = REP(d) + maxr[d] * He;
                j.rows = T.R[s];
                j.fan = T.size[s];
            }
            p.M = (int)T.R[s];
            p.H = He;
            p.K = s == 0 ? 0 : He;
            p.A = s == 0 ? nullptr : H(d) + prev;
            p.lda = He;
            p.A_hi = s == 0 ? nullptr : rep ? REP(d) : HI(d) + prev;
            p.A_lo = s == 0 ? nullptr : rep ? REP(d) + maxr[d] * He : LO(d) + prev;
            p.ldah = He;
            p.W = E.enc[d].W.as<float>();
            p.G = E.enc[d].G.as<float>();
            p.slot_ptr = T.digits.as<int>() + T.off[s];
            p.slot_stride = 1;
            p.slot_base = E.in_offset[(size_t)T.order[s]];
            p.c_prev = s == 0 ? nullptr : CB(d, s - 1);
            p.ldc_prev = He;
            p.parent = rep ? T.digits.as<int>() + T.total + T.off[s] : nullptr;
            p.c_out = CB(d, s);
            p.ldc = He;
            p.h_out = H(d) + cur;
            p.ldh = He;
            p.hA_hi = HI(d) + cur;
            p.hA_lo = LO(d) + cur;
            p.ldha = He;
            p.ha_bf16 = E.precision == KS_PREC_BF16 ? 1 : 0;
        }
        if (na == 0) continue;
        if (nr) {
            long long n = 0;
            for (int i = 0; i < nr; ++i) n = std::max(n, rj[i].rows * (long long)(He / 8));
            enc_prefix_replicate<<<dim3((unsigned)std::min<long long>((n + 255) / 256, 8LL * E.num_sms), (unsigned)nr),
                                   256, 0, E.stream>>>(rj[0], rj[1], He);
            E.launches++;
            KS_CUDA(cudaGetLastError());
        }
        double fl = 0.0;
        for (int i = 0; i < na; ++i) fl += s == 0 ? 0.0 : 2.0 * (double)a[i].M * He * 4.0 * He;
        if ((st = launch_lstm(E, a[0], na == 2 ? &a[1] : nullptr, E.enc[dd[0]], na == 2 ? &E.enc[1] : nullptr, fl)))
            return st;
    }
    EncGatherArgs g;
    std::memset(&g, 0, sizeof g);
    g.tok = d_tok;
    g.C = (int)C;
    g.He = He;
    for (int d = 0; d < 2; ++d) {
        const ks_engine::EncTable& T = E.etab[d];
        g.S[d] = covered[d];
        for (int j = 0; j < 7; ++j) {
            g.order[d][j] = T.order[j];
            g.size[d][j] = T.size[j];
            g.off[d][j] = T.off[j];
        }
        if (covered[d] < 0) continue;
        g.h[d] = H(d);
        g.hi[d] = HI(d);
        g.lo[d] = LO(d);
        g.c[d] = CB(d, covered[d]);
        g.c_last[d] = (covered[d] & 1) ? c_slot1 + (size_t)d * 2 * C * He : c_slot0 + (size_t)d * 2 * C * He;
    }
    g.act = act;
    g.ahi = ahi;
    g.alo = alo;
    g.act_ld = act_ld;
    g.NA2 = NA2;
    g.NA = E.NA;
    const long long warps = C * (long long)(g.S[0] + 1 + g.S[1] + 1);
    enc_prefix_gather<<<(unsigned)std::min<long long>((warps + 7) / 8, 16LL * E.num_sms), 256, 0, E.stream>>>(g);
    E.launches++;
    KS_CUDA(cudaGetLastError());
    return KS_OK;
}

// reuse_encoder: the chunk's encoder outputs (a_t, encoder state, P^T, hybrid
// features) from the previous run_chunk on the SAME tokens are still in the
// workspace -- decode again at another beam width without re-encoding
// (topk_metrics over several k, eval.cpp:74-152)
ks_status run_chunk(ks_engine& E, int64_t C, int64_t cfg_base, int k, bool greedy, const int* d_tok,
                    const long long* d_desc, const PredDev& pd, int* o_tok, double* o_lp,
                    int* o_count, int* o_status, int* o_fpred, int* o_fstep, bool reuse_encoder = false) {
    ks_status st;
    if ((st = ensure_workspace(E, C, k))) return st;
    cudaStream_t s = E.stream;
    const bool enc_dec = E.variant == KS_VARIANT_ENC_DEC;
    if (!reuse_encoder) {
        // small batches: 32-unit N tiles double the CTAs of every gate GEMM of the chunk
        // (the weights, P^T and every launch of a chunk use one tile width)
        const bool hyb = E.variant == KS_VARIANT_HYBRID2 || E.variant == KS_VARIANT_HYBRID;
        const DevLstm& ref = hyb ? E.hb1[0] : E.dec;
        const int64_t rows = C * (int64_t)std::max(1, k);
        const int64_t tiles64 = (rows + 127) / 128 * std::max(1, ref.H / 64);
        E.units_now = (E.tc_units == 64 && ref.Whi32.p != nullptr && tiles64 < E.num_sms) ? 32 : E.tc_units;
    }
    const bool split = E.precision != KS_PREC_FP32;
    const int He = enc_dec ? E.NE : E.NA;
    const int NA2 = enc_dec ? 0 : 2 * E.NA;
    const int Hd = enc_dec ? E.NE : E.NS;
    const int Kd = NA2 + Hd;
    const long long act_ld = enc_dec ? 0 : 7LL * NA2;
    float* act = E.act.as<float>();
    float* encc = E.encc.as<float>();
    __half* encA = E.encA.as<__half>();
    auto encc_at = [&](int dir, int pp) { return encc + ((size_t)dir * 2 + pp) * C * He; };
    auto encA_at = [&](int dir, int pp, int lo) { return encA + (((size_t)dir * 2 + pp) * 2 + lo) * C * He; };

    const bool hybrid = E.variant == KS_VARIANT_HYBRID2 || E.variant == KS_VARIANT_HYBRID;
    if (!reuse_encoder && hybrid && (st = encode_hybrid(E, C, d_tok))) return st;
    // ---- encoder (bi-LSTM over the 7 one-hot input steps, zero initial state)
    const int dirs = enc_dec ? 1 : 2;
    // steps with fewer token prefixes than the chunk has configs run per prefix
    int covered[2] = {-1, -1};
    if (!reuse_encoder && !hybrid && !enc_dec && split && E.ctxproj && (E.etab[0].S >= 0 || E.etab[1].S >= 0) &&
        (st = encode_prefix(E, C, d_tok, act, E.actA.as<__half>(), E.actA.as<__half>() + (size_t)C * 7 * NA2, act_ld,
                            NA2, encc_at(0, 0), encc_at(0, 1), covered)))
        return st;
    for (int sidx = 0; sidx < ((hybrid || reuse_encoder) ? 0 : 7); ++sidx) {
        LstmArgs a[2];
        for (int dir = 0; dir < dirs; ++dir) {
            const int t = dir == 0 ? sidx : 6 - sidx;
            const int tprev = dir == 0 ? t - 1 : t + 1;
            LstmArgs& p = a[dir];
            std::memset(&p, 0, sizeof p);
            p.M = (int)C;
            p.H = He;
            p.K = sidx == 0 ? 0 : He;
            if (enc_dec) {
                // hidden state ping-pongs through the split planes and a scratch fp32 copy
                p.A = act + (size_t)((sidx + 1) & 1) * C * He;
                p.lda = He;
                p.h_out = act + (size_t)(sidx & 1) * C * He;
                p.ldh = He;
            } else {
                p.A = act + (size_t)tprev * NA2 + dir * E.NA;
                p.lda = act_ld;
                p.h_out = act + (size_t)t * NA2 + dir * E.NA;
                p.ldh = act_ld;
            }
            // attn / attn-2 with the context projection: the encoder's split h goes
            // straight into the a_t operand planes of the projection GEMM (actA rows
            // b*7 + t, columns dir*NA..), and the next step reads its A operand there
            // (row stride 7*NA2) -- no separate split pass over a_t
            const bool to_actA = !enc_dec && split && E.ctxproj;
            __half* aAhi = to_actA ? E.actA.as<__half>() : nullptr;
            __half* aAlo = to_actA ? aAhi + (size_t)C * 7 * NA2 : nullptr;
            if (to_actA) {
                p.A_hi = aAhi + (size_t)tprev * NA2 + dir * E.NA;
                p.A_lo = aAlo + (size_t)tprev * NA2 + dir * E.NA;
                p.ldah = act_ld;
            } else {
                p.A_hi = encA_at(dir, (sidx + 1) & 1, 0);
                p.A_lo = encA_at(dir, (sidx + 1) & 1, 1);
            }
            p.W = E.enc[dir].W.as<float>();
            p.G = E.enc[dir].G.as<float>();
            p.slot_ptr = d_tok + t;
            p.slot_stride = 7;
            p.slot_base = E.in_offset[(size_t)t];
            p.c_prev = sidx == 0 ? nullptr : encc_at(dir, (sidx + 1) & 1);
            p.ldc_prev = He;
            p.parent = nullptr;
            p.c_out = encc_at(dir, sidx & 1);
            p.ldc = He;
            if (split && to_actA) {
                p.hA_hi = aAhi + (size_t)t * NA2 + dir * E.NA;
                p.hA_lo = aAlo + (size_t)t * NA2 + dir * E.NA;
                p.ldha = act_ld;
                p.ha_bf16 = E.precision == KS_PREC_BF16 ? 1 : 0;
            } else if (split) {
                p.hA_hi = encA_at(dir, sidx & 1, 0);
                p.hA_lo = encA_at(dir, sidx & 1, 1);
                p.ldha = He;
                p.ha_bf16 = E.precision == KS_PREC_BF16 ? 1 : 0;
            }
        }
        int act_dirs[2], na = 0;
        for (int dir = 0; dir < dirs; ++dir)
            if (sidx > covered[dir]) act_dirs[na++] = dir;
        if (na == 0) continue;
        const double fl = sidx == 0 ? 0.0 : 2.0 * na * (double)C * He * 4.0 * He;
        const int d0 = act_dirs[0];
        if ((st = launch_lstm(E, a[d0], na == 2 ? &a[1] : nullptr, E.enc[d0], na == 2 ? &E.enc[1] : nullptr, fl)))
            return st;
    }
    bool any_proj = false;
    for (int pos = 0, h = 1; pos < E.T; h = (int)std::min<int64_t>(k, (int64_t)h * E.vsize[(size_t)pos]), ++pos)
        any_proj = any_proj || E.proj_at(pos, h);
    if (any_proj && reuse_encoder && !E.pt_valid)
        return set_error(KS_ERR_STATE, "encoder reuse without a context projection in the workspace");
    if (any_proj && !reuse_encoder) {
        // context projection P[c][t] = a_t . W_ctx (the ctx rows of the post-LSTM weight),
        // one GEMM over the C*7 encoder activations; raw pre-activations, no bias / cell
        LstmArgs q{};
        q.M = (int)(C * 7);
        q.H = Hd;
        q.K = NA2;
        q.A = act;
        q.lda = NA2;
        __half* ahi = E.actA.as<__half>();  // written by the encoder steps (to_actA above)
        __half* alo = ahi + (size_t)C * 7 * NA2;
        q.A_hi = ahi;
        q.A_lo = alo;
        q.W = E.dec.W.as<float>();
        q.G = E.dec.G.as<float>();
        q.ldw = Kd;                  // tensor-core layout [4H][Kd]: columns 0..NA2 are the ctx rows
        q.wcol = 0;
        q.raw = 1;
        q.ldt = (C * 7 + 7) / 8 * 8;
        q.pt_hi = E.Pt.as<__half>();
        q.pt_lo = q.pt_hi + (size_t)4 * Hd * q.ldt;
        if ((st = launch_lstm(E, q, nullptr, E.dec, nullptr, 0.0))) return st;
    }
    if (!reuse_encoder) E.pt_valid = any_proj;
    beam_init<<<(unsigned)((C + 255) / 256), 256, 0, s>>>((int)C, E.live[0].as<unsigned char>(),
                                                          E.lp[0].as<double>(),
                                                          E.key[0].as<unsigned long long>(),
                                                          E.status.as<int>(), E.fpred.as<int>(),
                                                          E.fstep.as<int>());
    E.launches++;

    // ---- decoder positions
    float* hb = E.hbuf.as<float>();
    float* cb = E.cbuf.as<float>();
    const int64_t R = C * k;
    int H = 1;
    int maxc = 8;
    {
        int h = 1;
        for (int p = 0; p < E.T; ++p) {
            maxc = std::max(maxc, h * E.vsize[(size_t)p]);
            h = std::min<int64_t>(k, (int64_t)h * E.vsize[(size_t)p]);
        }
    }
    const int cpw = (maxc + 7) / 8 * 8;
    int vmax = 1;
    for (int p = 0; p < E.T; ++p) vmax = std::max(vmax, E.vsize[(size_t)p]);
    cudaEvent_t keys_ready = nullptr;
    if (pd.has_host) {
        if (!pd.hook) return set_error(KS_ERR_PARAMETER, "host predicates need ks_beam_search_batch_hooked");
        if (E.hk_keys.ensure((size_t)R * 8) || E.hk_live.ensure((size_t)R) ||
            E.hk_rej.ensure((size_t)R * vmax * 4) || E.hrej.ensure((size_t)R * vmax * 4))
            return set_error(KS_ERR_CUDA, "host-hook buffers");
        cudaEventCreateWithFlags(&keys_ready, cudaEventDisableTiming);
    }
    int alpha_fill_H = -1;  // rows-per-config of the alpha-block layout currently in A_hi/lo
    for (int pos = 0; pos < E.T; ++pos) {
        const int cur = pos & 1, nxt = cur ^ 1;
        const int M = (int)(C * H);
        if (pd.has_host) {
            // live prefixes of this position leave the device now; the hook runs on the
            // host while the GPU computes this position's attention and gate GEMM
            KS_CUDA(cudaMemcpyAsync(E.hk_keys.p, E.key[cur].p, (size_t)M * 8, cudaMemcpyDeviceToHost, s));
            KS_CUDA(cudaMemcpyAsync(E.hk_live.p, E.live[cur].p, (size_t)M, cudaMemcpyDeviceToHost, s));
            KS_CUDA(cudaEventRecord(keys_ready, s));
        }
        // previous position's state (or the initial state at position 0)
        const float* h_prev = nullptr;
        const float* c_prev = nullptr;
        const int* par = nullptr;
        if (pos > 0) {
            h_prev = hb + (size_t)((pos - 1) & 1) * R * Hd;
            c_prev = cb + (size_t)((pos - 1) & 1) * R * Hd;
            par = E.parent[cur].as<int>();
        } else if (enc_dec) {
            h_prev = act + (size_t)(6 & 1) * C * He;   // encoder final state (thought vector)
            c_prev = encc_at(0, 6 & 1);
            par = nullptr;                              // H_0 = 1: row r = config r
        }
        // position 1: every hypothesis is a child of the single root (H_0 = 1), and
        // siblings share [ctx | h_prev] and c_prev -- attention and the gate GEMM run
        // once per config (classic ctx operand) and the GEMM epilogue fans each
        // parent row's gates out to its H children (gates + G[slot(child)])
        const bool fan_ok = pos == 1 && H > 1 && !enc_dec && !hybrid && E.precision != KS_PREC_FP32 &&
                            E.ctxproj && !E.pair_now();
        // with compaction on, position 1 runs as a compacted position (one parent per
        // config, classic [ctx | h] operand) on the 16-warp compacted epilogue
        const bool cp1 = fan_ok && E.compact && E.compact_pos1;
        const bool fan = fan_ok && !cp1;
        const int Mg = fan ? (int)C : M;  // rows of this position's attention and gate GEMM
        // positions >= 2 (alpha blocks): attention and the gate GEMM run on each config's
        // distinct live parents (compacted rows, 128-row tiles), the GEMM epilogue writes
        // their children
        const bool compact = cp1 || (E.compact && pos >= 2 && !fan && H > 1 && !enc_dec && !hybrid &&
                                     E.precision != KS_PREC_FP32 && E.proj_at(pos, H) && !E.pair_now());
        int *cp_cnt = nullptr, *cp_base = nullptr, *cp_cfg = nullptr, *cp_prow = nullptr, *cp_cst = nullptr,
            *cp_ccn = nullptr;
        int4* cp_child = nullptr;
        const int kal_c = E.alpha_cols_for(128, 1);  // <= 128 configs per 128-row tile
        if (compact) {
            cp_cnt = E.cpbuf.as<int>();
            cp_base = cp_cnt + C;
            cp_cfg = cp_base + C + 2;
            cp_prow = cp_cfg + M;
            cp_cst = cp_prow + M;
            cp_ccn = cp_cst + M;
            cp_child = reinterpret_cast<int4*>(
                (reinterpret_cast<uintptr_t>(cp_ccn + M) + 15) & ~static_cast<uintptr_t>(15));
            const unsigned g = (unsigned)((C + 255) / 256);
            const int* slots = E.variant == KS_VARIANT_ATTN2 ? nullptr : E.slot[cur].as<int>();
            cp_count<<<g, 256, 0, s>>>(par, E.live[cur].as<unsigned char>(), (int)C, H, cp_cnt, cp_base);
            cp_fill<<<g, 256, 0, s>>>(par, E.live[cur].as<unsigned char>(), slots, (int)C, H, cp_cnt, cp_base,
                                      cp_base + C, cp_cfg, cp_prow, cp_cst, cp_ccn, cp_child);
            E.launches += 2;
            KS_CUDA(cudaGetLastError());
        }
        AttnArgs aa{};
        aa.M = Mg;
        aa.H_rows = fan ? 1 : H;
        aa.NS = Hd;
        aa.NA2 = NA2;
        aa.nd = E.n_d;
        aa.h_prev = h_prev;
        aa.ldh = Hd;
        aa.parent = fan ? nullptr : par;  // fan: row b of position 0 is config b's root
        aa.act = act;
        aa.uatt = E.uatt.as<float>();
        aa.Ws = enc_dec ? nullptr : E.attWs.as<float>();
        aa.wo = enc_dec ? nullptr : E.attWo.as<float>();
        aa.Wa = enc_dec ? nullptr : E.attWa.as<float>();
        aa.bh = enc_dec ? nullptr : E.attBh.as<float>();
        aa.uatt_out = E.uatt.as<float>();
        aa.bo = E.attBo;
        aa.A = E.Abuf.as<float>();
        aa.A_hi = E.Ahi.as<__half>();
        aa.A_lo = E.Alo.as<__half>();
        aa.split_mode = E.precision == KS_PREC_FP32 ? 0 : (E.precision == KS_PREC_F16X3 ? 1 : 2);
        aa.kalpha = (!fan && E.proj_at(pos, H)) ? E.alpha_cols_of(H) : 0;
        aa.alpha_tile = E.alpha_tile_of(H);
        // same rows and layout as the previous alpha-block position: its zeros are still in place
        aa.alpha_sparse = (aa.kalpha && alpha_fill_H == H) ? 1 : 0;
        alpha_fill_H = aa.kalpha ? H : -1;
        if (compact) {
            aa.kalpha = cp1 ? 0 : kal_c;
            aa.alpha_tile = 128;
            aa.alpha_sparse = 0;
            alpha_fill_H = -1;  // the next position rewrites its layout in full
            aa.cp_M = cp_base + C;
            aa.cp_cfg = cp_cfg;
            aa.cp_prow = cp_prow;
        }
        if (enc_dec) aa.nd = 0;
        if (!hybrid) {
            if (!launch_attention(aa, pos == 0 && !enc_dec, s))
                return set_error(KS_ERR_UNSUPPORTED, "attention_dense_nodes outside 1..8");
            E.launches++;
        }

        LstmArgs p{};
        p.M = Mg;
        p.H = Hd;
        p.K = Kd;
        p.A = E.Abuf.as<float>();
        p.lda = Kd;
        p.A_hi = E.Ahi.as<__half>();
        p.A_lo = E.Alo.as<__half>();
        p.W = E.dec.W.as<float>();
        p.G = E.dec.G.as<float>();
        if (E.variant == KS_VARIANT_ATTN2) {
            p.slot_ptr = nullptr;
            p.slot_base = 0;
        } else if (pos == 0) {
            p.slot_ptr = nullptr;
            p.slot_base = 0;     // GO token, feedback slot 0 (encoding.cpp:192-199)
        } else {
            p.slot_ptr = E.slot[cur].as<int>();
            p.slot_stride = 1;
            p.slot_base = 0;
        }
        p.c_prev = c_prev;
        p.ldc_prev = Hd;
        p.parent = fan ? nullptr : par;
        p.fan = fan ? H : 0;
        p.h_out = hb + (size_t)cur * R * Hd;
        p.ldh = Hd;
        p.c_out = cb + (size_t)cur * R * Hd;
        p.ldc = Hd;
        if (enc_dec && pos == 0) p.ldc_prev = He;
        if (E.ctxproj && pos == 0) {
            // h = 0 at position 0: contract the ctx columns only
            p.K = NA2;
            p.ldah = Kd;
            p.ldw = Kd;
            p.wcol = 0;
        } else if (cp1) {
            // position 1 compacted: classic [ctx | h_prev] rows of the roots
            p.parent = nullptr;
            p.alpha_tile = 128;
            p.cp_M = cp_base + C;
            p.cp_cfg = cp_cfg;
            p.cp_prow = cp_prow;
            p.cp_cstart = cp_cst;
            p.cp_ccount = cp_ccn;
            p.cp_child = cp_child;
        } else if (!fan && E.proj_at(pos, H)) {
            // [alpha block | h_prev] . [P^T | W_h]  (ctx . W_ctx = sum_t alpha_t P_t)
            const int kal = E.alpha_cols_of(H);
            p.K = kal + Hd;
            p.ldah = 0;
            p.ldw = Kd;
            p.wcol = NA2;
            p.kb_alpha = kal / kTcBK;
            p.rows_per_cfg = H;
            p.alpha_tile = E.alpha_tile_of(H);
            p.PT_hi = E.Pt.as<__half>();
            p.ldpt = (C * 7 + 7) / 8 * 8;
            p.PT_lo = p.PT_hi + (size_t)4 * Hd * p.ldpt;
            p.pt_rows = C * 7;
            if (compact) {
                p.K = kal_c + Hd;
                p.kb_alpha = kal_c / kTcBK;
                p.alpha_tile = 128;
                p.parent = nullptr;
                p.cp_M = cp_base + C;
                p.cp_cfg = cp_cfg;
                p.cp_prow = cp_prow;
                p.cp_cstart = cp_cst;
                p.cp_ccount = cp_ccn;
                p.cp_child = cp_child;
            }
        }
        const double useful = 2.0 * (double)M * (double)(2 * E.n_a * (enc_dec ? 0 : 1) + (enc_dec ? E.e : E.n_s)) *
                              4.0 * (enc_dec ? E.e : E.n_s);
        if (!hybrid && (st = launch_lstm(E, p, nullptr, E.dec, nullptr, useful))) return st;
        const int* host_rej = nullptr;
        if (pd.has_host) {
            KS_CUDA(cudaEventSynchronize(keys_ready));
            const int V = E.vsize[(size_t)pos];
            const unsigned long long* keys = E.hk_keys.as<unsigned long long>();
            const unsigned char* live = E.hk_live.as<unsigned char>();
            int* rej = E.hk_rej.as<int>();
            std::vector<int32_t> rcfg, rpre, rout;
            std::vector<int64_t> ridx;
            for (int64_t r = 0; r < M; ++r) {
                for (int v = 0; v < V; ++v) rej[r * V + v] = -1;
                if (!live[r]) continue;
                ridx.push_back(r);
                rcfg.push_back((int32_t)(cfg_base + r / H));
                for (int t = 0; t < pos; ++t)
                    rpre.push_back((int32_t)((keys[r] >> E.meta.shift[t]) & ((1ull << E.meta.bits[t]) - 1ull)));
            }
            rout.assign(ridx.size() * (size_t)V, -1);
            if (!ridx.empty() &&
                pd.hook(pd.user, pos, pos == E.T - 1 ? 1 : 0, (int64_t)ridx.size(), rcfg.data(),
                        rpre.empty() ? nullptr : rpre.data(), V, rout.data()) != 0) {
                cudaEventDestroy(keys_ready);
                return set_error(KS_ERR_STATE, "host predicate hook aborted the search");
            }
            for (size_t i = 0; i < ridx.size(); ++i)
                for (int v = 0; v < V; ++v) rej[ridx[i] * V + v] = rout[i * V + v];
            KS_CUDA(cudaMemcpyAsync(E.hrej.p, rej, (size_t)M * V * 4, cudaMemcpyHostToDevice, s));
            host_rej = E.hrej.as<int>();
        }

        const int V = E.vsize[(size_t)pos];
        const bool fin = pos == E.T - 1;
        const int Hn = fin ? 0 : (int)std::min<int64_t>(k, (int64_t)H * V);
        BeamArgs b{};
        b.B = (int)C;
        b.H_cur = H;
        b.H_next = Hn;
        b.pos = pos;
        b.k = k;
        b.greedy = greedy ? 1 : 0;
        b.final_step = fin ? 1 : 0;
        b.NS = hybrid ? 2 * E.CP : Hd;
        b.h = hybrid ? E.feat.as<float>() + (size_t)pos * C * 2 * E.CP : hb + (size_t)cur * R * Hd;
        b.h_per_config = hybrid ? 1 : 0;
        b.Wh = E.headW[(size_t)pos]->as<float>();
        b.bh = E.headB[(size_t)pos]->as<float>();
        b.live_cur = E.live[cur].as<unsigned char>();
        b.lp_cur = E.lp[cur].as<double>();
        b.key_cur = E.key[cur].as<unsigned long long>();
        b.live_next = E.live[nxt].as<unsigned char>();
        b.lp_next = E.lp[nxt].as<double>();
        b.key_next = E.key[nxt].as<unsigned long long>();
        b.parent_next = E.parent[nxt].as<int>();
        b.slot_next = E.slot[nxt].as<int>();
        b.status = E.status.as<int>();
        b.fail_pred = E.fpred.as<int>();
        b.fail_step = E.fstep.as<int>();
        b.preds = E.preds.as<DevPred>();
        b.n_preds = pd.n;
        b.pred_bytes = E.pbytes.as<unsigned char>();
        b.term_pos = E.tpos.as<int>();
        b.term_w = E.tw.as<double>();
        b.term_field = E.tfield.as<int>();
        b.values = E.values.as<long long>();
        b.desc = d_desc;
        b.out_tok = o_tok;
        b.out_lp = o_lp;
        b.out_count = o_count;
        b.out_status = o_status;
        b.out_fail_pred = o_fpred;
        b.out_fail_step = o_fstep;
        b.cands_per_warp = cpw;
        b.host_rej = host_rej;
        b.n_values = (int)E.out_values.size();
        b.n_terms = pd.n_terms;
        b.n_bytes = pd.n_bytes;
        if (E.fw_dist) {  // model_forward (ks_forward_batch): greedy, one row per config
            b.teacher = E.fw_teacher;
            b.out_dist = E.fw_dist;
            b.dist_ld = E.fw_ld;
            int off = 0;
            for (int q = 0; q < pos; ++q) off += E.vsize[(size_t)q];
            b.dist_off = off;
        }
        const size_t tables = (size_t)b.n_values * 8 + (size_t)b.n_terms * 16 + (size_t)pd.n * sizeof(DevPred) +
                              (size_t)b.n_bytes + 16;
        int warps = 8;
        while (warps > 1 && beam_smem_bytes(b.NS, V, warps, cpw, tables) > (size_t)E.beam_smem_max) --warps;
        const size_t smem = beam_smem_bytes(b.NS, V, warps, cpw, tables);
        if (smem > (size_t)E.beam_smem_max)
            return set_error(KS_ERR_UNSUPPORTED, "beam width x vocabulary too large for the beam kernel");
        // persistent: the head weights are staged into shared memory once per CTA
        // upper bound (one warp per config); launch_beam trims it to one resident wave
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((C + warps - 1) / warps, (int64_t)E.num_sms * 16));
        if (!launch_beam(b, E.meta, warps, smem, grid, s))
            return set_error(KS_ERR_CUDA, "beam kernel launch failed");
        E.launches++;
        const cudaError_t err = cudaGetLastError();
        if (err != cudaSuccess) return set_error(KS_ERR_CUDA, std::string("beam launch: ") + cudaGetErrorString(err));
        if (E.debug_parents && pos + 1 < E.T) {  // diagnostic (KS_DEBUG_PARENTS=1): synchronous
            if (E.dbg.ensure(16)) return set_error(KS_ERR_CUDA, "debug counter allocation failed");
            cudaMemsetAsync(E.dbg.p, 0, 16, s);
            dbg_parents<<<(unsigned)((C + 255) / 256), 256, 0, s>>>(E.parent[nxt].as<int>(),
                                                                    E.live[nxt].as<unsigned char>(), (int)C, Hn,
                                                                    E.dbg.as<unsigned long long>());
            unsigned long long hv[2];
            cudaMemcpyAsync(hv, E.dbg.p, 16, cudaMemcpyDeviceToHost, s);
            cudaStreamSynchronize(s);
            fprintf(stderr, "pos %d -> %d: rows/config %d, live %.3f, distinct parents %.3f\n", pos, pos + 1, Hn,
                    (double)hv[1] / C, (double)hv[0] / C);
        }
        H = Hn;
    }
    if (keys_ready) {
        cudaStreamSynchronize(s);  // pinned host-hook buffers are reused by the next chunk
        cudaEventDestroy(keys_ready);
    }
    return KS_OK;
}

// run_chunk through a cached CUDA graph: one launch replays the whole decode of a
// chunk (tens of kernels), removing the per-kernel launch gaps that dominate
// small batches.  Not used with host predicates (host round trips), profiling
// (events) or when disabled.
ks_status run_chunk_graph(ks_engine& E, int64_t C, int64_t cfg_base, int k, bool greedy, const int* d_tok,
                          const long long* d_desc, const PredDev& pd, int* o_tok, double* o_lp, int* o_count,
                          int* o_status, int* o_fpred, int* o_fstep, bool single_chunk) {
    // multi-chunk decodes through caller buffers would cycle through one graph per chunk
    // offset: plain launches (decode_chunks passes its two internal buffer sets instead)
    if (!single_chunk || !E.use_graphs || E.prof || pd.has_host)
        return run_chunk(E, C, cfg_base, k, greedy, d_tok, d_desc, pd, o_tok, o_lp, o_count, o_status, o_fpred,
                         o_fstep);
    ks_status st;
    if ((st = ensure_workspace(E, C, k))) return st;  // allocations before the key is taken
    auto P = [](const void* p) { return (long long)reinterpret_cast<uintptr_t>(p); };
    // cfg_base only reaches the host-hook rows, and host predicates bypass graphs: a
    // chunk at any offset replays the graph of its buffers
    const std::vector<long long> key = {C, k, greedy ? 1 : 0, P(d_tok), P(d_desc), pd.n, pd.n_terms,
                                        pd.n_bytes, pd.needs_desc ? 1 : 0, P(o_tok), P(o_lp), P(o_count),
                                        P(o_status), P(o_fpred), P(o_fstep),
                                        (long long)g_alloc_gen.load()};
    for (auto& g : E.graphs)
        if (g.key == key) {
            KS_CUDA(cudaGraphLaunch(g.exec, E.stream));
            E.launches += g.launches;
            return KS_OK;
        }
    const int64_t l0 = E.launches;
    // a capture that fails (an operation the driver refuses inside a capture) turns
    // graphs off for this engine and the chunk runs as plain launches
    auto plain = [&]() {
        (void)cudaGetLastError();
        E.use_graphs = false;
        E.launches = l0;
        return run_chunk(E, C, cfg_base, k, greedy, d_tok, d_desc, pd, o_tok, o_lp, o_count, o_status, o_fpred,
                         o_fstep);
    };
    if (cudaStreamBeginCapture(E.stream, cudaStreamCaptureModeRelaxed) != cudaSuccess) return plain();
    st = run_chunk(E, C, cfg_base, k, greedy, d_tok, d_desc, pd, o_tok, o_lp, o_count, o_status, o_fpred, o_fstep);
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(E.stream, &graph);
    if (st || ce != cudaSuccess || !graph) {
        if (graph) cudaGraphDestroy(graph);
        return plain();
    }
    cudaGraphExec_t exec = nullptr;
    const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ie != cudaSuccess) return plain();
    if (E.graphs.size() >= 8) {
        cudaGraphExecDestroy(E.graphs.front().exec);
        E.graphs.erase(E.graphs.begin());
    }
    E.graphs.push_back({key, exec, E.launches - l0});
    KS_CUDA(cudaGraphLaunch(exec, E.stream));
    return KS_OK;
}

ks_status check_common(ks_engine* eng, int64_t B, int32_t k, const ks_pred* preds, int32_t n) {
    if (!eng) return set_error(KS_ERR_PARAMETER, "null engine");
    if (k < 1) return set_error(KS_ERR_PARAMETER, "beam width must be >= 1, got " + std::to_string(k));
    if (B < 0) return set_error(KS_ERR_PARAMETER, "negative batch size");
    if (n < 0 || (n > 0 && !preds)) return set_error(KS_ERR_PARAMETER, "bad predicate list");
    if (cudaSetDevice(eng->device) != cudaSuccess) return set_error(KS_ERR_CUDA, "cudaSetDevice failed");
    return KS_OK;
}

ks_status collect_profile(ks_engine& E) {
    for (size_t i = 0; i < E.prof_ev.size(); ++i) {
        float ms = 0.0f;
        cudaEventSynchronize(E.prof_ev[i].second);
        cudaEventElapsedTime(&ms, E.prof_ev[i].first, E.prof_ev[i].second);
        E.prof_ms += ms;
        E.prof_useful += E.prof_flops[i];
        E.prof_n++;
        E.prof_each.emplace_back(ms, E.prof_flops[i]);
        E.prof_each_exec.push_back(E.prof_exec[i]);
        cudaEventDestroy(E.prof_ev[i].first);
        cudaEventDestroy(E.prof_ev[i].second);
    }
    E.prof_ev.clear();
    E.prof_flops.clear();
    E.prof_exec.clear();
    return KS_OK;
}

// Host-side copies of the reference-facing call (pageable <-> pinned staging):
// large ones are split over a few threads (one memcpy thread reaches ~10 GB/s).
void par_memcpy(void* dst, const void* src, size_t bytes) {
    constexpr size_t kPart = (size_t)2 << 20;
    const int parts = (int)std::min<size_t>(8, bytes / kPart);
    if (parts < 2) {
        std::memcpy(dst, src, bytes);
        return;
    }
    const size_t step = (bytes / parts + 63) / 64 * 64;
    std::vector<std::thread> th;
    for (int i = 1; i < parts; ++i) {
        const size_t o = (size_t)i * step;
        if (o >= bytes) break;
        th.emplace_back([=] { std::memcpy((char*)dst + o, (const char*)src + o, std::min(step, bytes - o)); });
    }
    std::memcpy(dst, src, std::min(step, bytes));
    for (auto& t : th) t.join();
}

// Where a decode call's inputs come from and its results go.
struct ChunkOut {
    int32_t* tok;
    double* lp;
    int32_t* count;
    int32_t* status;
    int32_t* fpred;
    int32_t* fstep;
};

// The chunk pipeline behind every batch decode.  B configs run in chunks of C =
// E.chunk; chunk i uses buffer set s = i & 1:
//   stream:       [inputs -> io[s].tok]  wait(copy_done[s])  decode (CUDA graph)  record dec_done[s]
//   copy_stream:  wait(dec_done[s])  results io[s] -> caller (D2H / D2D)  record copy_done[s]
//   host:         stage chunk i's inputs; unpack chunk i-1's results (staged D2H)
// so chunk i's decode overlaps chunk i-1's result transfer and host unpacking, and
// every chunk replays one of (at most) three graphs: full chunk in set 0 / 1, the
// tail chunk.  device_io: tok / desc / outputs are device pointers and `user` is the
// caller's stream (ordered before and after the call by events); otherwise host
// buffers, page-locked results receiving the D2H copy directly.
ks_status decode_chunks(ks_engine& E, int64_t B, int k, bool greedy, const PredDev& pd, const int32_t* tok,
                        const int64_t* desc, bool device_io, int32_t* out_tok, double* out_lp, int32_t* out_count,
                        int32_t* out_status, int32_t* out_fpred, int32_t* out_fstep, cudaStream_t user) {
    const int T = E.T;
    E.launches = 0;
    const int64_t C = std::max<int64_t>(1, std::min<int64_t>(B, E.chunk));
    const bool want_desc = desc && pd.needs_desc;
    for (auto& b : E.io) {
        if (b.tok.ensure((size_t)C * 7 * 4) || (want_desc && b.desc.ensure((size_t)C * 7 * 8)) ||
            b.otok.ensure((size_t)C * k * T * 4) || b.olp.ensure((size_t)C * k * 8) ||
            b.ocount.ensure((size_t)C * 4) || b.ostatus.ensure((size_t)C * 4) || b.ofpred.ensure((size_t)C * 4) ||
            b.ofstep.ensure((size_t)C * 4))
            return set_error(KS_ERR_CUDA, "chunk buffer allocation failed");
        if (!device_io && (b.h_in.ensure((size_t)C * 7 * 4 + (size_t)C * 7 * 8) ||
                           b.h_out.ensure((size_t)C * k * T * 4 + (size_t)C * k * 8 + (size_t)C * 4 * 4)))
            return set_error(KS_ERR_CUDA, "pinned staging allocation failed");
    }
    ks_status st;
    if ((st = ensure_workspace(E, C, k))) return st;
    cudaStream_t s = E.stream, cs = E.copy_stream;
    if (device_io) {  // the caller's prior work (inputs) before ours
        KS_CUDA(cudaEventRecord(E.io[1].dec_done, user));
        KS_CUDA(cudaStreamWaitEvent(s, E.io[1].dec_done, 0));
    }
    // page-locked host results take the device-to-host copy directly
    auto pinned = [](const void* p) {
        if (!p) return true;
        cudaPointerAttributes a{};
        const bool ok = cudaPointerGetAttributes(&a, p) == cudaSuccess && a.type == cudaMemoryTypeHost;
        (void)cudaGetLastError();
        return ok;
    };
    const bool direct = device_io || (pinned(out_tok) && (greedy || (pinned(out_lp) && pinned(out_count) &&
                                                                    pinned(out_status) && pinned(out_fpred) &&
                                                                    pinned(out_fstep))));
    const cudaMemcpyKind out_kind = device_io ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    // host side of a staged chunk: pinned staging -> caller buffers
    auto unpack = [&](int sb, int64_t c0, int64_t n) -> ks_status {
        KS_CUDA(cudaEventSynchronize(E.io[sb].copy_done));
        if (direct) return KS_OK;
        const char* ho = E.io[sb].h_out.as<char>();
        const int32_t* h_tok = reinterpret_cast<const int32_t*>(ho);
        const double* h_lp = reinterpret_cast<const double*>(ho + (size_t)C * k * T * 4);
        const int32_t* h_misc = reinterpret_cast<const int32_t*>(ho + (size_t)C * k * T * 4 + (size_t)C * k * 8);
        par_memcpy(out_tok + c0 * k * T, h_tok, (size_t)n * k * T * 4);
        if (!greedy) {
            if (out_lp) par_memcpy(out_lp + c0 * k, h_lp, (size_t)n * k * 8);
            if (out_count) std::memcpy(out_count + c0, h_misc, (size_t)n * 4);
            if (out_status) std::memcpy(out_status + c0, h_misc + C, (size_t)n * 4);
            if (out_fpred) std::memcpy(out_fpred + c0, h_misc + 2 * C, (size_t)n * 4);
            if (out_fstep) std::memcpy(out_fstep + c0, h_misc + 3 * C, (size_t)n * 4);
        }
        return KS_OK;
    };
    int64_t prev_c0 = -1, prev_n = 0;
    int prev_sb = 0;
    for (int64_t c0 = 0, i = 0; c0 < B; c0 += C, ++i) {
        const int64_t n = std::min<int64_t>(C, B - c0);
        const int sb = (int)(i & 1);
        auto& b = E.io[sb];
        // inputs of this chunk (the staging of set sb was last read by chunk i - 2's
        // upload, which completed before its results were unpacked)
        const long long* ddesc = nullptr;
        if (device_io) {
            KS_CUDA(cudaMemcpyAsync(b.tok.p, tok + c0 * 7, (size_t)n * 7 * 4, cudaMemcpyDeviceToDevice, s));
            if (want_desc)
                KS_CUDA(cudaMemcpyAsync(b.desc.p, desc + c0 * 7, (size_t)n * 7 * 8, cudaMemcpyDeviceToDevice, s));
        } else {
            int32_t* htok = b.h_in.as<int32_t>();
            par_memcpy(htok, tok + c0 * 7, (size_t)n * 7 * 4);
            KS_CUDA(cudaMemcpyAsync(b.tok.p, htok, (size_t)n * 7 * 4, cudaMemcpyHostToDevice, s));
            if (want_desc) {
                int64_t* hdesc = reinterpret_cast<int64_t*>(b.h_in.as<char>() + (size_t)C * 7 * 4);
                std::memcpy(hdesc, desc + c0 * 7, (size_t)n * 7 * 8);
                KS_CUDA(cudaMemcpyAsync(b.desc.p, hdesc, (size_t)n * 7 * 8, cudaMemcpyHostToDevice, s));
            }
        }
        if (want_desc) ddesc = b.desc.as<long long>();
        // the decode overwrites set sb's results: chunk i - 2's copy-out must be done
        KS_CUDA(cudaStreamWaitEvent(s, b.copy_done, 0));
        if ((st = run_chunk_graph(E, n, c0, k, greedy, b.tok.as<int>(), ddesc, pd, b.otok.as<int>(),
                                  b.olp.as<double>(), b.ocount.as<int>(), b.ostatus.as<int>(), b.ofpred.as<int>(),
                                  b.ofstep.as<int>(), true)))
            return st;
        KS_CUDA(cudaEventRecord(b.dec_done, s));
        KS_CUDA(cudaStreamWaitEvent(cs, b.dec_done, 0));
        if (direct) {
            KS_CUDA(cudaMemcpyAsync(out_tok + c0 * k * T, b.otok.p, (size_t)n * k * T * 4, out_kind, cs));
            if (!greedy) {
                if (out_lp) KS_CUDA(cudaMemcpyAsync(out_lp + c0 * k, b.olp.p, (size_t)n * k * 8, out_kind, cs));
                if (out_count) KS_CUDA(cudaMemcpyAsync(out_count + c0, b.ocount.p, (size_t)n * 4, out_kind, cs));
                if (out_status) KS_CUDA(cudaMemcpyAsync(out_status + c0, b.ostatus.p, (size_t)n * 4, out_kind, cs));
                if (out_fpred) KS_CUDA(cudaMemcpyAsync(out_fpred + c0, b.ofpred.p, (size_t)n * 4, out_kind, cs));
                if (out_fstep) KS_CUDA(cudaMemcpyAsync(out_fstep + c0, b.ofstep.p, (size_t)n * 4, out_kind, cs));
            }
        } else {
            char* ho = b.h_out.as<char>();
            int32_t* h_misc = reinterpret_cast<int32_t*>(ho + (size_t)C * k * T * 4 + (size_t)C * k * 8);
            KS_CUDA(cudaMemcpyAsync(ho, b.otok.p, (size_t)n * k * T * 4, cudaMemcpyDeviceToHost, cs));
            if (!greedy) {
                KS_CUDA(cudaMemcpyAsync(ho + (size_t)C * k * T * 4, b.olp.p, (size_t)n * k * 8, cudaMemcpyDeviceToHost, cs));
                KS_CUDA(cudaMemcpyAsync(h_misc, b.ocount.p, (size_t)n * 4, cudaMemcpyDeviceToHost, cs));
                KS_CUDA(cudaMemcpyAsync(h_misc + C, b.ostatus.p, (size_t)n * 4, cudaMemcpyDeviceToHost, cs));
                KS_CUDA(cudaMemcpyAsync(h_misc + 2 * C, b.ofpred.p, (size_t)n * 4, cudaMemcpyDeviceToHost, cs));
                KS_CUDA(cudaMemcpyAsync(h_misc + 3 * C, b.ofstep.p, (size_t)n * 4, cudaMemcpyDeviceToHost, cs));
            }
        }
        KS_CUDA(cudaEventRecord(b.copy_done, cs));
        // the previous chunk's results, unpacked while this chunk decodes
        if (!device_io && prev_c0 >= 0 && (st = unpack(prev_sb, prev_c0, prev_n))) return st;
        prev_c0 = c0;
        prev_n = n;
        prev_sb = sb;
    }
    if (device_io) {  // the caller's stream continues after our last copy
        if (prev_c0 >= 0) KS_CUDA(cudaStreamWaitEvent(user, E.io[prev_sb].copy_done, 0));
    } else if (prev_c0 >= 0 && (st = unpack(prev_sb, prev_c0, prev_n))) {
        return st;
    }
    if (E.prof) collect_profile(E);
    return KS_OK;
}

ks_status decode_host(ks_engine* eng, const int32_t* tok, const int64_t* desc, int64_t B, int32_t k,
                      bool greedy, const ks_pred* preds, int32_t n_preds, int32_t* out_tok,
                      double* out_lp, int32_t* out_count, int32_t* out_status, int32_t* out_fpred,
                      int32_t* out_fstep, ks_host_pred_fn hook = nullptr, void* user = nullptr) {
    ks_engine& E = *eng;
    const int T = E.T;
    {
        uint32_t lim[7];
        for (int f = 0; f < 7; ++f) lim[f] = (uint32_t)E.in_sizes[(size_t)f];
        bool bad = false;
        for (int64_t b = 0; b < B && !bad; ++b) {
            const int32_t* r = tok + b * 7;
            bad = ((uint32_t)r[0] >= lim[0]) | ((uint32_t)r[1] >= lim[1]) | ((uint32_t)r[2] >= lim[2]) |
                  ((uint32_t)r[3] >= lim[3]) | ((uint32_t)r[4] >= lim[4]) | ((uint32_t)r[5] >= lim[5]) |
                  ((uint32_t)r[6] >= lim[6]);
        }
        if (bad)
            for (int64_t b = 0; b < B; ++b)
                for (int f = 0; f < 7; ++f) {
                    const int t = tok[b * 7 + f];
                    if (t < 0 || t >= E.in_sizes[(size_t)f])
                        return set_error(KS_ERR_INDEX, "input token " + std::to_string(t) + " out of range for field " +
                                                           std::to_string(f) + " (row " + std::to_string(b) + ")");
                }
    }
    PredDev pd;
    ks_status st;
    if ((st = upload_preds(E, preds, n_preds, pd))) return st;
    if (pd.needs_desc && !desc) return set_error(KS_ERR_PARAMETER, "divisibility predicates need descriptors");
    pd.hook = hook;
    pd.user = user;
    return decode_chunks(E, B, k, greedy, pd, tok, desc, /*device_io=*/false, out_tok, out_lp, out_count,
                         out_status, out_fpred, out_fstep, nullptr);
}

}  // namespace

extern "C" ks_status ks_beam_search_batch(ks_engine* eng, const int32_t* tok, const int64_t* desc,
                                          int64_t B, int32_t k, const ks_pred* preds, int32_t n_preds,
                                          int32_t* out_tok, double* out_lp, int32_t* out_count,
                                          int32_t* out_status, int32_t* out_fpred, int32_t* out_fstep) {
    if (!eng) return set_error(KS_ERR_PARAMETER, "null engine");
    std::lock_guard<std::mutex> lock(eng->mu);
    ks_status st = check_common(eng, B, k, preds, n_preds);
    if (st) return st;
    if (B == 0) return KS_OK;
    if (!tok || !out_tok) return set_error(KS_ERR_PARAMETER, "null token buffer");
    return decode_host(eng, tok, desc, B, k, false, preds, n_preds, out_tok, out_lp, out_count, out_status,
                       out_fpred, out_fstep);
}

extern "C" ks_status ks_beam_search_batch_hooked(ks_engine* eng, const int32_t* tok, const int64_t* desc,
                                                 int64_t B, int32_t k, const ks_pred* preds, int32_t n_preds,
                                                 ks_host_pred_fn hook, void* user, int32_t* out_tok,
                                                 double* out_lp, int32_t* out_count, int32_t* out_status,
                                                 int32_t* out_fpred, int32_t* out_fstep) {
    if (!eng) return set_error(KS_ERR_PARAMETER, "null engine");
    std::lock_guard<std::mutex> lock(eng->mu);
    ks_status st = check_common(eng, B, k, preds, n_preds);
    if (st) return st;
    if (B == 0) return KS_OK;
    if (!tok || !out_tok) return set_error(KS_ERR_PARAMETER, "null token buffer");
    return decode_host(eng, tok, desc, B, k, false, preds, n_preds, out_tok, out_lp, out_count, out_status,
                       out_fpred, out_fstep, hook, user);
}

extern "C" ks_status ks_topk_metrics_batch(ks_engine* eng, const int32_t* tok, const int64_t* desc,
                                           const int32_t* truth, int64_t B, int32_t k, const ks_pred* preds,
                                           int32_t n_preds, ks_host_pred_fn hook, void* user,
                                           int64_t* out_pos_matches, int64_t* out_perfect) {
    if (!eng) return set_error(KS_ERR_PARAMETER, "null engine");
    std::lock_guard<std::mutex> lock(eng->mu);
    ks_status st = check_common(eng, B, k, preds, n_preds);
    if (st) return st;
    if (!tok || !truth || !out_pos_matches || !out_perfect) return set_error(KS_ERR_PARAMETER, "null buffer");
    ks_engine& E = *eng;
    const int T = E.T;
    for (int p = 0; p < T; ++p) out_pos_matches[p] = 0;
    *out_perfect = 0;
    if (B == 0) return KS_OK;
    for (int64_t b = 0; b < B; ++b)
        for (int p = 0; p < T; ++p) {
            const int v = truth[b * T + p];
            if (v < 0 || v >= E.vsize[(size_t)p])
                return set_error(KS_ERR_INDEX, "truth token " + std::to_string(v) + " out of range at position " +
                                                   std::to_string(p) + " (row " + std::to_string(b) + ")");
        }
    for (int64_t b = 0; b < B; ++b)
        for (int f = 0; f < 7; ++f) {
            const int t = tok[b * 7 + f];
            if (t < 0 || t >= E.in_sizes[(size_t)f])
                return set_error(KS_ERR_INDEX, "input token " + std::to_string(t) + " out of range for field " +
                                                   std::to_string(f) + " (row " + std::to_string(b) + ")");
        }
    PredDev pd;
    if ((st = upload_preds(E, preds, n_preds, pd))) return st;
    if (pd.needs_desc && !desc) return set_error(KS_ERR_PARAMETER, "divisibility predicates need descriptors");
    pd.hook = hook;
    pd.user = user;
    E.launches = 0;
    const int64_t C = std::max<int64_t>(1, std::min<int64_t>(B, E.chunk));
    if (E.otok.ensure((size_t)C * k * T * 4) || E.olp.ensure((size_t)C * k * 8) || E.ocount.ensure((size_t)C * 4) ||
        E.ostatus.ensure((size_t)C * 4) || E.ofpred.ensure((size_t)C * 4) || E.ofstep.ensure((size_t)C * 4) ||
        E.truth.ensure((size_t)C * T * 4) || E.evalc.ensure((size_t)(T + 1) * 8))
        return set_error(KS_ERR_CUDA, "output allocation failed");
    if ((st = ensure_workspace(E, C, k))) return st;
    KS_CUDA(cudaMemsetAsync(E.evalc.p, 0, (size_t)(T + 1) * 8, E.stream));
    for (int64_t c0 = 0; c0 < B; c0 += C) {
        const int64_t n = std::min<int64_t>(C, B - c0);
        KS_CUDA(cudaMemcpyAsync(E.tok.p, tok + c0 * 7, (size_t)n * 7 * 4, cudaMemcpyHostToDevice, E.stream));
        KS_CUDA(cudaMemcpyAsync(E.truth.p, truth + c0 * T, (size_t)n * T * 4, cudaMemcpyHostToDevice, E.stream));
        const long long* ddesc = nullptr;
        if (desc && pd.needs_desc) {
            KS_CUDA(cudaMemcpyAsync(E.desc.p, desc + c0 * 7, (size_t)n * 7 * 8, cudaMemcpyHostToDevice, E.stream));
            ddesc = E.desc.as<long long>();
        }
        if ((st = run_chunk(E, n, c0, k, false, E.tok.as<int>(), ddesc, pd, E.otok.as<int>(), E.olp.as<double>(),
                            E.ocount.as<int>(), E.ostatus.as<int>(), E.ofpred.as<int>(), E.ofstep.as<int>())))
            return st;
        unsigned long long* cnt = E.evalc.as<unsigned long long>();
        if (!launch_topk_eval(E.otok.as<int>(), E.ocount.as<int>(), E.truth.as<int>(), (int)n, k, T, cnt, cnt + T,
                              E.stream))
            return set_error(KS_ERR_CUDA, "topk_eval launch failed");
        E.launches++;
    }
    std::vector<unsigned long long> h((size_t)T + 1);
    KS_CUDA(cudaMemcpyAsync(h.data(), E.evalc.p, (size_t)(T + 1) * 8, cudaMemcpyDeviceToHost, E.stream));
    KS_CUDA(cudaStreamSynchronize(E.stream));
    for (int p = 0; p < T; ++p) out_pos_matches[p] = (int64_t)h[(size_t)p];
    *out_perfect = (int64_t)h[(size_t)T];
    if (E.prof) collect_profile(E);
    return KS_OK;
}

extern "C" ks_status ks_topk_metrics_multi(ks_engine* eng, const int32_t* tok, const int64_t* desc,
                                           const int32_t* truth, int64_t B, const int32_t* k_values, int32_t n_k,
                                           const ks_pred* preds, int32_t n_preds, ks_host_pred_fn hook, void* user,
                                           int64_t* out_pos_matches, int64_t* out_perfect) {
    if (!eng) return set_error(KS_ERR_PARAMETER, "null engine");
    if (!k_values || n_k < 1) return set_error(KS_ERR_PARAMETER, "no beam widths");
    int kmax = 0;
    for (int i = 0; i < n_k; ++i) {
        if (k_values[i] < 1) return set_error(KS_ERR_PARAMETER, "beam width must be >= 1");
        kmax = std::max(kmax, (int)k_values[i]);
    }
    std::lock_guard<std::mutex> lock(eng->mu);
    ks_status st = check_common(eng, B, kmax, preds, n_preds);
    if (st) return st;
    if (!tok || !truth || !out_pos_matches || !out_perfect) return set_error(KS_ERR_PARAMETER, "null buffer");
    ks_engine& E = *eng;
    const int T = E.T;
    for (int64_t i = 0; i < (int64_t)n_k * T; ++i) out_pos_matches[i] = 0;
    for (int i = 0; i < n_k; ++i) out_perfect[i] = 0;
    if (B == 0) return KS_OK;
    for (int64_t b = 0; b < B; ++b)
        for (int p = 0; p < T; ++p) {
            const int v = truth[b * T + p];
            if (v < 0 || v >= E.vsize[(size_t)p])
                return set_error(KS_ERR_INDEX, "truth token " + std::to_string(v) + " out of range at position " +
                                                   std::to_string(p) + " (row " + std::to_string(b) + ")");
        }
    for (int64_t b = 0; b < B; ++b)
        for (int f = 0; f < 7; ++f) {
            const int t = tok[b * 7 + f];
            if (t < 0 || t >= E.in_sizes[(size_t)f])
                return set_error(KS_ERR_INDEX, "input token " + std::to_string(t) + " out of range for field " +
                                                   std::to_string(f) + " (row " + std::to_string(b) + ")");
        }
    PredDev pd;
    if ((st = upload_preds(E, preds, n_preds, pd))) return st;
    if (pd.needs_desc && !desc) return set_error(KS_ERR_PARAMETER, "divisibility predicates need descriptors");
    pd.hook = hook;
    pd.user = user;
    E.launches = 0;
    // widest first: its encoding fixes the chunk's GEMM tile width and computes the
    // context projection every narrower width may use
    std::vector<int> order((size_t)n_k);
    for (int i = 0; i < n_k; ++i) order[(size_t)i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return k_values[a] > k_values[b]; });
    const int64_t C = std::max<int64_t>(1, std::min<int64_t>(B, E.chunk));
    if (E.otok.ensure((size_t)C * kmax * T * 4) || E.olp.ensure((size_t)C * kmax * 8) ||
        E.ocount.ensure((size_t)C * 4) || E.ostatus.ensure((size_t)C * 4) || E.ofpred.ensure((size_t)C * 4) ||
        E.ofstep.ensure((size_t)C * 4) || E.truth.ensure((size_t)C * T * 4) ||
        E.evalc.ensure((size_t)n_k * (T + 1) * 8))
        return set_error(KS_ERR_CUDA, "output allocation failed");
    if ((st = ensure_workspace(E, C, kmax))) return st;  // no reallocation between the widths
    KS_CUDA(cudaMemsetAsync(E.evalc.p, 0, (size_t)n_k * (T + 1) * 8, E.stream));
    unsigned long long* cnt = E.evalc.as<unsigned long long>();
    for (int64_t c0 = 0; c0 < B; c0 += C) {
        const int64_t n = std::min<int64_t>(C, B - c0);
        KS_CUDA(cudaMemcpyAsync(E.tok.p, tok + c0 * 7, (size_t)n * 7 * 4, cudaMemcpyHostToDevice, E.stream));
        KS_CUDA(cudaMemcpyAsync(E.truth.p, truth + c0 * T, (size_t)n * T * 4, cudaMemcpyHostToDevice, E.stream));
        const long long* ddesc = nullptr;
        if (desc && pd.needs_desc) {
            KS_CUDA(cudaMemcpyAsync(E.desc.p, desc + c0 * 7, (size_t)n * 7 * 8, cudaMemcpyHostToDevice, E.stream));
            ddesc = E.desc.as<long long>();
        }
        for (size_t oi = 0; oi < order.size(); ++oi) {
            const int i = order[oi];
            const int k = k_values[i];
            if ((st = run_chunk(E, n, c0, k, false, E.tok.as<int>(), ddesc, pd, E.otok.as<int>(), E.olp.as<double>(),
                                E.ocount.as<int>(), E.ostatus.as<int>(), E.ofpred.as<int>(), E.ofstep.as<int>(),
                                oi > 0)))
                return st;
            unsigned long long* ci = cnt + (size_t)i * (T + 1);
            if (!launch_topk_eval(E.otok.as<int>(), E.ocount.as<int>(), E.truth.as<int>(), (int)n, k, T, ci, ci + T,
                                  E.stream))
                return set_error(KS_ERR_CUDA, "topk_eval launch failed");
            E.launches++;
        }
    }
    std::vector<unsigned long long> h((size_t)n_k * (T + 1));
    KS_CUDA(cudaMemcpyAsync(h.data(), E.evalc.p, h.size() * 8, cudaMemcpyDeviceToHost, E.stream));
    KS_CUDA(cudaStreamSynchronize(E.stream));
    for (int i = 0; i < n_k; ++i) {
        for (int p = 0; p < T; ++p) out_pos_matches[(size_t)i * T + p] = (int64_t)h[(size_t)i * (T + 1) + p];
        out_perfect[i] = (int64_t)h[(size_t)i * (T + 1) + T];
    }
    if (E.prof) collect_profile(E);
    return KS_OK;
}

extern "C" ks_status ks_host_register(void* p, int64_t bytes) {
    if (!p || bytes <= 0) return set_error(KS_ERR_PARAMETER, "null or empty host buffer");
    const cudaError_t e = cudaHostRegister(p, (size_t)bytes, cudaHostRegisterDefault);
    if (e == cudaErrorHostMemoryAlreadyRegistered) {
        (void)cudaGetLastError();
        return KS_OK;
    }
    if (e != cudaSuccess) return set_error(KS_ERR_CUDA, std::string("cudaHostRegister: ") + cudaGetErrorString(e));
    return KS_OK;
}

extern "C" ks_status ks_host_unregister(void* p) {
    if (!p) return set_error(KS_ERR_PARAMETER, "null host buffer");
    const cudaError_t e = cudaHostUnregister(p);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        return set_error(KS_ERR_CUDA, std::string("cudaHostUnregister: ") + cudaGetErrorString(e));
    }
    return KS_OK;
}

extern "C" ks_status ks_greedy_batch(ks_engine* eng, const int32_t* tok, int64_t B, int32_t* out_tok) {
    if (!eng) return set_error(KS_ERR_PARAMETER, "null engine");
    std::lock_guard<std::mutex> lock(eng->mu);
    ks_status st = check_common(eng, B, 1, nullptr, 0);
    if (st) return st;
    if (B == 0) return KS_OK;
    if (!tok || !out_tok) return set_error(KS_ERR_PARAMETER, "null token buffer");
    return decode_host(eng, tok, nullptr, B, 1, true, nullptr, 0, out_tok, nullptr, nullptr, nullptr, nullptr,
                       nullptr);
}

extern "C" ks_status ks_forward_batch(ks_engine* eng, const int32_t* tok, const int32_t* teacher, int64_t B,
                                      double* out_dist, int32_t* out_tok, double* out_score) {
    if (!eng) return set_error(KS_ERR_PARAMETER, "null engine");
    std::lock_guard<std::mutex> lock(eng->mu);
    if (B < 0 || B > (1LL << 31)) return set_error(KS_ERR_PARAMETER, "batch size out of range");
    if (B == 0) return KS_OK;
    if (!tok || !out_dist) return set_error(KS_ERR_PARAMETER, "null buffer");
    ks_engine& E = *eng;
    cudaSetDevice(E.device);
    const int T = E.T;
    int SV = 0;
    for (int q = 0; q < T; ++q) SV += E.vsize[(size_t)q];
    for (int64_t b = 0; b < B; ++b)
        for (int f = 0; f < 7; ++f) {
            const int t = tok[b * 7 + f];
            if (t < 0 || t >= E.in_sizes[(size_t)f])
                return set_error(KS_ERR_INDEX, "input token " + std::to_string(t) + " out of range for field " +
                                                   std::to_string(f) + " (row " + std::to_string(b) + ")");
        }
    if (teacher)
        for (int64_t b = 0; b < B; ++b)
            for (int q = 0; q < T; ++q) {
                const int t = teacher[b * T + q];
                if (t < 0 || t >= E.vsize[(size_t)q])
                    return set_error(KS_ERR_INDEX, "teacher token " + std::to_string(t) + " out of range at position " +
                                                       std::to_string(q) + " (row " + std::to_string(b) + ")");
            }
    PredDev pd;
    ks_status st;
    if ((st = upload_preds(E, nullptr, 0, pd))) return st;
    E.launches = 0;
    const int64_t C = std::max<int64_t>(1, std::min<int64_t>(B, E.chunk));
    if (E.otok.ensure((size_t)C * T * 4) || E.olp.ensure((size_t)C * 8) || E.ocount.ensure((size_t)C * 4) ||
        E.fwd.ensure((size_t)C * SV * 8) || (teacher && E.fwt.ensure((size_t)C * T * 4)) ||
        E.tok.ensure((size_t)C * 7 * 4))
        return set_error(KS_ERR_CUDA, "forward buffers");
    if ((st = ensure_workspace(E, C, 1))) return st;
    struct Reset {  // the forward hooks never outlive this call
        ks_engine& e;
        ~Reset() {
            e.fw_teacher = nullptr;
            e.fw_dist = nullptr;
        }
    } reset{E};
    E.fw_teacher = teacher ? E.fwt.as<int>() : nullptr;
    E.fw_dist = E.fwd.as<double>();
    E.fw_ld = SV;
    std::vector<int32_t> tk;
    for (int64_t c0 = 0; c0 < B; c0 += C) {
        const int64_t n = std::min<int64_t>(C, B - c0);
        KS_CUDA(cudaMemcpyAsync(E.tok.p, tok + c0 * 7, (size_t)n * 7 * 4, cudaMemcpyHostToDevice, E.stream));
        if (teacher)
            KS_CUDA(cudaMemcpyAsync(E.fwt.p, teacher + c0 * T, (size_t)n * T * 4, cudaMemcpyHostToDevice, E.stream));
        if ((st = run_chunk(E, n, c0, 1, true, E.tok.as<int>(), nullptr, pd, E.otok.as<int>(), E.olp.as<double>(),
                            E.ocount.as<int>(), nullptr, nullptr, nullptr)))
            return st;
        KS_CUDA(cudaMemcpyAsync(out_dist + c0 * SV, E.fwd.p, (size_t)n * SV * 8, cudaMemcpyDeviceToHost, E.stream));
        if (out_tok)
            KS_CUDA(cudaMemcpyAsync(out_tok + c0 * T, E.otok.p, (size_t)n * T * 4, cudaMemcpyDeviceToHost, E.stream));
        if (out_score)
            KS_CUDA(cudaMemcpyAsync(out_score + c0, E.olp.p, (size_t)n * 8, cudaMemcpyDeviceToHost, E.stream));
        KS_CUDA(cudaStreamSynchronize(E.stream));
    }
    return KS_OK;
}

extern "C" ks_status ks_beam_search_device(ks_engine* eng, const int32_t* d_tok, const int64_t* d_desc,
                                           int64_t B, int32_t k, const ks_pred* preds, int32_t n_preds,
                                           int32_t* d_out_tok, double* d_out_lp, int32_t* d_out_count,
                                           int32_t* d_out_status, int32_t* d_out_fpred,
                                           int32_t* d_out_fstep, void* stream) {
    if (!eng) return set_error(KS_ERR_PARAMETER, "null engine");
    std::lock_guard<std::mutex> lock(eng->mu);
    ks_status st = check_common(eng, B, k, preds, n_preds);
    if (st) return st;
    if (B == 0) return KS_OK;
    if (!d_tok || !d_out_tok || !d_out_lp || !d_out_count)
        return set_error(KS_ERR_PARAMETER, "null device buffer");
    ks_engine& E = *eng;
    PredDev pd;
    if ((st = upload_preds(E, preds, n_preds, pd))) return st;
    if (pd.needs_desc && !d_desc) return set_error(KS_ERR_PARAMETER, "divisibility predicates need descriptors");
    return decode_chunks(E, B, k, false, pd, d_tok, d_desc, /*device_io=*/true, d_out_tok, d_out_lp, d_out_count,
                         d_out_status, d_out_fpred, d_out_fstep, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" void ks_engine_profile_reset(ks_engine* eng, int32_t enable) {
    if (!eng) return;
    collect_profile(*eng);
    eng->prof = enable != 0;
    eng->prof_ms = 0.0;
    eng->prof_useful = 0.0;
    eng->prof_n = 0;
    eng->prof_each.clear();
    eng->prof_each_exec.clear();
}

extern "C" int64_t ks_engine_profile_launches(const ks_engine* eng, int64_t cap, double* ms, double* useful) {
    if (!eng) return 0;
    const int64_t n = (int64_t)eng->prof_each.size();
    for (int64_t i = 0; i < n && i < cap; ++i) {
        if (ms) ms[i] = eng->prof_each[(size_t)i].first;
        if (useful) useful[i] = eng->prof_each[(size_t)i].second;
    }
    return n;
}

extern "C" int64_t ks_engine_profile_launches_ex(const ks_engine* eng, int64_t cap, double* ms, double* useful,
                                                 double* mma_issued) {
    if (!eng) return 0;
    const int64_t n = ks_engine_profile_launches(eng, cap, ms, useful);
    for (int64_t i = 0; i < n && i < cap && mma_issued; ++i) mma_issued[i] = eng->prof_each_exec[(size_t)i];
    return n;
}

extern "C" double ks_engine_profile_gemm_ms(const ks_engine* eng, int64_t* launches, double* useful) {
    if (!eng) return 0.0;
    if (launches) *launches = eng->prof_n;
    if (useful) *useful = eng->prof_useful;
    return eng->prof_ms;
}
