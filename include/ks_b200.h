/* ks_b200.h -- the drop-in C-ABI of the B200 constrained-beam-decode engine.
 *
 * Plain C types only (no torch, no C++).  Everything the reference's
 * `kernelseer` C++/Python API needs for the hot path -- model load, encode,
 * greedy / beam / constrained beam search over a batch of problem
 * descriptors, predicate registration -- crosses this boundary.  The C++
 * host layer (include/kernelseer_b200/*.hpp) and the Python module are
 * written on top of it; INTEGRATION.md shows the bindings a maintainer of
 * the reference would add.
 *
 * Reference interfaces replaced (paths under /root/reference/proj):
 *   ks_checkpoint_*            load_checkpoint          src/data.cpp:513-665, include/kernelseer/data.hpp:77
 *   ks_engine_create           SequencePredictor ctor   src/models.cpp:377-379, include/kernelseer/models.hpp:80-98
 *   ks_encode_problems         encode_problem           src/encoding.cpp:87-113, include/kernelseer/encoding.hpp:80-81
 *   ks_beam_search_batch       beam_search /            src/decoding.cpp:27-103, 126-135
 *                              constrained_beam_search  include/kernelseer/decoding.hpp:28-36
 *   ks_greedy_batch            greedy_decode            src/decoding.cpp:107-124, include/kernelseer/decoding.hpp:23-24
 *   ks_forward_batch           model_forward /          src/models.cpp:495-514, 387-493,
 *                              SequencePredictor::step  include/kernelseer/models.hpp:80-103
 *   ks_pred (typed programs)   ConstraintPredicate +    include/kernelseer/constraints.hpp:45-63,
 *                              membership_predicate /   src/constraints.cpp:198-242
 *                              resource_budget_predicate
 *   ks_status                  exception taxonomy       include/kernelseer/errors.hpp:10-87
 *   ks_trainer_*               train_model batch body,  src/models.cpp:788-797, 827-856, 905-947,
 *                              model_loss_gradients,    src/nn.cpp:262-297
 *                              evaluate_set, adam_step
 *   the batch entry points     parallel_stripes fan-out include/kernelseer/parallel.hpp:14-27 as used
 *                              in topk_metrics          src/eval.cpp:105-137
 *   ks_topk_metrics_batch      topk_metrics scoring     src/eval.cpp:100-146
 *   ks_engine_group_*, ks_group_*  parallel_stripes     include/kernelseer/parallel.hpp:14-27,
 *                              (multi-GPU sharding)     src/eval.cpp:105-137
 */
#ifndef KS_B200_H
#define KS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One status code per reference exception class (errors.hpp). */
typedef enum {
    KS_OK = 0,
    KS_ERR_SHAPE = 1,          /* ShapeError */
    KS_ERR_PARAMETER = 2,      /* ParameterError (beam width < 1, bad sizes, ...) */
    KS_ERR_INDEX = 3,          /* IndexError (token id out of range) */
    KS_ERR_STATE = 4,          /* StateError (missing tensor, stepping past the end) */
    KS_ERR_VALIDATION = 5,     /* ValidationError (out-of-vocabulary descriptor field) */
    KS_ERR_CHECKPOINT = 6,     /* CheckpointError; see ks_checkpoint_error_kind */
    KS_ERR_BEAM_EXHAUSTED = 7, /* BeamExhaustedError (single-config calls only; batch calls
                                  report exhaustion per row in out_status) */
    KS_ERR_CUDA = 8,           /* device / driver failure */
    KS_ERR_UNSUPPORTED = 9     /* model variant or shape this engine does not implement */
} ks_status;

/* Thread-local message for the last non-OK status returned on this thread. */
const char* ks_last_error(void);
/* For KS_ERR_VALIDATION: the offending field name (ValidationError::field). */
const char* ks_last_error_field(void);

/* ------------------------------------------------------------------------- */
/* Checkpoint: kernelseer-checkpoint/1 (docs/formats.md:53-93)                */
/* ------------------------------------------------------------------------- */
typedef struct ks_checkpoint ks_checkpoint;

/* CheckpointError kinds (errors.hpp:66-74): 0 version, 1 truncated, 2 shape,
 * 3 malformed, 4 io. */
ks_status ks_checkpoint_load(const char* path, ks_checkpoint** out);
int32_t ks_checkpoint_error_kind(void);
void ks_checkpoint_free(ks_checkpoint* ck);
/* Header value by key ("variant", "kernel", "post_attention_size", ...); NULL if absent. */
const char* ks_checkpoint_header(const ks_checkpoint* ck, const char* key);
int32_t ks_checkpoint_num_tensors(const ks_checkpoint* ck);
/* i-th tensor in payload (= alphabetical) order: name, rank, dims[3], fp32 data. */
ks_status ks_checkpoint_tensor(const ks_checkpoint* ck, int32_t i, const char** name,
                               int32_t* rank, int32_t* dims, const float** data);

/* ------------------------------------------------------------------------- */
/* Model description for engine creation (the fields of ModelParams,         */
/* models.hpp:45-53, flattened).                                              */
/* ------------------------------------------------------------------------- */
enum { KS_VARIANT_ENC_DEC = 0, KS_VARIANT_ATTN = 1, KS_VARIANT_ATTN2 = 2,
       KS_VARIANT_HYBRID = 3, KS_VARIANT_HYBRID2 = 4 };

typedef struct {
    int32_t variant;              /* KS_VARIANT_* (ModelVariant, models.hpp:16) */
    int32_t encoder_state_size;   /* |e| */
    int32_t pre_attention_size;   /* n_a (per direction) */
    int32_t post_attention_size;  /* n_s */
    int32_t attention_dense_nodes;/* n_d */
    int32_t num_positions;        /* T_out */
    const int32_t* input_sizes;   /* 7 input-field vocabulary sizes (order n,c,h,w,k,y,x) */
    const int64_t* input_values;  /* concatenated input values, ascending per field */
    const int32_t* vocab_sizes;   /* T_out output-parameter vocabulary sizes */
    const int64_t* output_values; /* concatenated output values in spec order */
    int32_t num_tensors;
    const char* const* tensor_names; /* reference names: "post.w_input", "head.3.bias", ... */
    const int32_t* tensor_numel;
    const float* const* tensor_data; /* fp32 (checkpoints are fp32, data.cpp:447-460) */
    /* hybrid variants (models.hpp:22-41): conv stack and bi-LSTM cell size */
    int32_t decoder_cell_size;
    int32_t num_conv_layers;
    const int32_t* conv_layers;      /* num_conv_layers x (filters, kernel_size, stride) */
} ks_model_desc;

/* Arithmetic of the gate GEMMs (the 99.6% of FLOPs):
 *   KS_PREC_F16X3: tcgen05 tensor cores, fp16 hi/lo operand split with three
 *                  MMAs (hi*hi + hi*lo + lo*hi), fp32 accumulate in TMEM --
 *                  fp32-grade accuracy; the default and the parity path.
 *   KS_PREC_FP32:  CUDA-core fp32 FFMA (exact fp32 GEMM); a second parity path.
 *   KS_PREC_BF16:  tcgen05 single bf16 MMA, fp32 accumulate -- reduced precision,
 *                  reported as decoded-sequence agreement. */
enum { KS_PREC_F16X3 = 0, KS_PREC_FP32 = 1, KS_PREC_BF16 = 2 };

/* An engine owns its weights and one device workspace: calls on the same
 * engine are serialized by an internal lock (safe from several threads, as the
 * reference's read-only SequencePredictor is); create one engine per GPU /
 * stream for concurrent decoding.  A ks_trainer is single-threaded. */
typedef struct ks_engine ks_engine;

ks_status ks_engine_create(const ks_model_desc* model, int32_t device, int32_t precision,
                           ks_engine** out);
ks_status ks_engine_create_from_checkpoint(const char* path, int32_t device, int32_t precision,
                                           ks_engine** out);
void ks_engine_destroy(ks_engine* eng);

int32_t ks_engine_num_positions(const ks_engine* eng);
int32_t ks_engine_vocab_size(const ks_engine* eng, int32_t position);
int32_t ks_engine_precision(const ks_engine* eng);
/* Number of kernel launches issued by the last decode call (evidence for bench). */
int64_t ks_engine_last_launch_count(const ks_engine* eng);
/* Configs per internal chunk (device workspace is sized for it); 0 = default. */
ks_status ks_engine_set_chunk(ks_engine* eng, int64_t configs_per_chunk);

/* encode_problem for B descriptors (B x 7 int64, field order n,c,h,w,k,y,x):
 * writes B x 7 token ids.  allow_nearest snaps unknown values (FieldVocab::nearest,
 * encoding.cpp:26-34).  On an unknown value returns KS_ERR_VALIDATION naming
 * the field of the first failing row; *bad_row receives its index. */
ks_status ks_encode_problems(const ks_engine* eng, const int64_t* desc, int64_t B,
                             int32_t allow_nearest, int32_t* tok, int64_t* bad_row);

/* Synthetic problem descriptors (benchmark / parity workloads):
 * config start+i (i < count) draws each of the 7 input fields uniformly with
 * replacement from the vocabulary (input_sizes[7], input_values concatenated per
 * field), one Rng::uniform_int per field in order n,c,h,w,k,y,x, from its own
 * stream Rng::derive(seed, start + i) (rng.hpp:19-43).  out_desc: count x 7.
 * The reference's generate_synthetic (data.cpp:348-395) draws unique grid
 * points and cannot produce 64k / 1M configs; no other reference counterpart. */
ks_status ks_synthetic_descriptors(const int32_t* input_sizes, const int64_t* input_values,
                                   uint64_t seed, int64_t start, int64_t count, int64_t* out_desc);
/* The same over an engine's model input vocabulary. */
ks_status ks_engine_synthetic_descriptors(const ks_engine* eng, uint64_t seed, int64_t start,
                                          int64_t count, int64_t* out_desc);

/* ------------------------------------------------------------------------- */
/* Typed predicate programs.  ConstraintPredicate::fn is an opaque callable in  */
/* the reference (constraints.hpp:49); the engine evaluates these typed forms */
/* on the device.  Registration order = evaluation order; the first rejecting */
/* predicate discards the candidate (decoding.cpp:69-76).                     */
/* ------------------------------------------------------------------------- */
enum {
    KS_PRED_MASK = 1,     /* allowed[value_offset(p) + token] for every assigned position:
                             membership_predicate and other per-value tables */
    KS_PRED_BUDGET = 2,   /* resource_budget_predicate: cost = sum over terms (ALPHABETICAL
                             parameter-name order) of w * value for assigned params, fp64
                             with separate multiply and add; accept iff cost <= budget */
    KS_PRED_PRODUCT = 3,  /* scale * prod(values of assigned listed params) <= limit
                             (workgroup size, LDS bytes); no reference counterpart */
    KS_PRED_DIVIDES = 4,  /* each assigned listed param value v > 0 divides the descriptor
                             field term_field[i] (tile divisibility); no reference counterpart */
    KS_PRED_HOST = 5      /* opaque host predicate (a reference std::function / Python callable):
                             evaluated by the ks_host_pred_fn hook between positions, in
                             registration order with the typed ones */
};

typedef struct {
    int32_t kind;
    int32_t full_sequence_only;   /* evaluate only at the last position (decoding.cpp:67-70) */
    const uint8_t* allowed;       /* MASK: sum_p vocab_size(p) entries */
    int32_t n_terms;
    const int32_t* term_pos;      /* output position per term; -1 = never assigned */
    const double* term_w;         /* BUDGET weights, terms in alphabetical name order */
    const int32_t* term_field;    /* DIVIDES descriptor field per term (0..6) */
    double budget;                /* BUDGET */
    int64_t scale;                /* PRODUCT */
    int64_t limit;                /* PRODUCT */
} ks_pred;

/* ------------------------------------------------------------------------- */
/* Decode.  Host-pointer entry points (the reference-facing call; copies are  */
/* part of the call).  tok: B x 7 token ids; desc: B x 7 descriptor values,   */
/* only read by KS_PRED_DIVIDES (may be NULL otherwise).                      */
/* Outputs: out_tok B x k x T (rank order, -1 padded), out_lp B x k (fp64),   */
/* out_count B (beams returned), out_status B (0 ok, 1 exhausted),            */
/* out_fail_pred / out_fail_step B (BeamExhaustedError::predicate index and   */
/* step, -1 when ok).  Any output pointer except out_tok may be NULL.          */
/* ------------------------------------------------------------------------- */
ks_status ks_beam_search_batch(ks_engine* eng, const int32_t* tok, const int64_t* desc,
                               int64_t B, int32_t beam_width, const ks_pred* preds,
                               int32_t n_preds, int32_t* out_tok, double* out_lp,
                               int32_t* out_count, int32_t* out_status,
                               int32_t* out_fail_pred, int32_t* out_fail_step);

/* Host hook for KS_PRED_HOST entries.  Called once per position (before that
 * position's selection) with the n_rows live hypotheses of the call: their
 * config index (0..B-1) and prefix tokens (n_rows x position, row-major).  For
 * every (row, token < vocab) it writes the registration index (into the
 * ks_pred array) of the first KS_PRED_HOST predicate that rejects the child,
 * or -1.  The device combines it with the typed predicates so the first
 * rejecting predicate in registration order wins (decoding.cpp:69-76).
 * The hook runs on the calling thread while the GPU computes the position's
 * attention and gate GEMM.  Return nonzero to abort the call. */
typedef int32_t (*ks_host_pred_fn)(void* user, int32_t position, int32_t final_step,
                                   int64_t n_rows, const int32_t* row_config,
                                   const int32_t* row_prefix, int32_t vocab,
                                   int32_t* out_first_reject);

/* ks_beam_search_batch with a host predicate hook (required when any
 * predicate has kind KS_PRED_HOST). */
ks_status ks_beam_search_batch_hooked(ks_engine* eng, const int32_t* tok, const int64_t* desc,
                                      int64_t B, int32_t beam_width, const ks_pred* preds,
                                      int32_t n_preds, ks_host_pred_fn hook, void* user,
                                      int32_t* out_tok, double* out_lp, int32_t* out_count,
                                      int32_t* out_status, int32_t* out_fail_pred,
                                      int32_t* out_fail_step);

/* topk_metrics' inner loop on the device (src/eval.cpp:100-146): a beam
 * search of width k over B configs (predicates / hook as
 * ks_beam_search_batch_hooked; hook may be NULL), then per config the
 * best-matching beam against truth (B x T token ids; most matching positions,
 * ties to the higher-ranked beam) and the any-of-k perfect flag, reduced on the
 * device.  out_pos_matches (T): per-position hits of the best-matching beams;
 * out_perfect: configs with a perfect beam.  Exhausted configs score nothing
 * (eval.cpp:114-116). */
ks_status ks_topk_metrics_batch(ks_engine* eng, const int32_t* tok, const int64_t* desc,
                                const int32_t* truth, int64_t B, int32_t beam_width,
                                const ks_pred* preds, int32_t n_preds, ks_host_pred_fn hook,
                                void* user, int64_t* out_pos_matches, int64_t* out_perfect);
/* topk_metrics over several beam widths (eval.cpp:74-152 runs one search per
 * k): each chunk is encoded ONCE (bi-LSTM / conv encoder and the context
 * projection) and decoded at every width, widest first; results identical to
 * n_k ks_topk_metrics_batch calls.  out_pos_matches: n_k x T, out_perfect: n_k,
 * both in k_values order. */
ks_status ks_topk_metrics_multi(ks_engine* eng, const int32_t* tok, const int64_t* desc,
                                const int32_t* truth, int64_t B, const int32_t* k_values, int32_t n_k,
                                const ks_pred* preds, int32_t n_preds, ks_host_pred_fn hook,
                                void* user, int64_t* out_pos_matches, int64_t* out_perfect);

/* greedy_decode: out_tok B x T. */
ks_status ks_greedy_batch(ks_engine* eng, const int32_t* tok, int64_t B, int32_t* out_tok);

/* model_forward (models.cpp:495-514) for B inputs at once: the decoder runs
 * greedily over all T positions, feeding back teacher[b][p] (B x T token ids)
 * when teacher != NULL, else its own argmax (lowest index on ties).
 *   out_dist  B x sum_p V_p: each position's softmax distribution (nn.cpp:215-226)
 *   out_tok   B x T (optional): the tokens fed back (teacher or argmax)
 *   out_score B (optional): sum_p log(max(dist_p[tok_p], 1e-300)), the
 *             teacher-forced sequence score of decoding_test.cpp:38-46
 * Also the device half of SequencePredictor::encode / initial_state / step
 * (models.hpp:80-98) in the C++ and Python layers. */
ks_status ks_forward_batch(ks_engine* eng, const int32_t* tok, const int32_t* teacher, int64_t B,
                           double* out_dist, int32_t* out_tok, double* out_score);

/* Page-lock (cudaHostRegister) / release a caller buffer.  Result buffers of the
 * host-buffer calls above that are page-locked receive the device-to-host copy
 * directly (no staging copy); callers reusing result buffers call by call
 * register them once.  No reference counterpart (a B200-side addition). */
ks_status ks_host_register(void* p, int64_t bytes);
ks_status ks_host_unregister(void* p);

/* Device-resident variant: every pointer is device memory; runs on `stream`
 * (a cudaStream_t, NULL = legacy default) and returns without synchronising. */
ks_status ks_beam_search_device(ks_engine* eng, const int32_t* d_tok, const int64_t* d_desc,
                                int64_t B, int32_t beam_width, const ks_pred* preds,
                                int32_t n_preds, int32_t* d_out_tok, double* d_out_lp,
                                int32_t* d_out_count, int32_t* d_out_status,
                                int32_t* d_out_fail_pred, int32_t* d_out_fail_step,
                                void* stream);

/* ------------------------------------------------------------------------- */
/* Engine groups: one engine per GPU, a batch sharded across them.  Replaces   */
/* parallel_stripes (parallel.hpp:14-27) as used by topk_metrics              */
/* (eval.cpp:105-137): configs are independent, so each device decodes a      */
/* contiguous balanced shard [g*B/G, (g+1)*B/G) on its own host thread and    */
/* writes its slice of the caller's outputs -- no collective, config order    */
/* preserved.  Outputs and errors are those of the single-engine calls; a     */
/* host predicate hook sees the caller's config indices and may be called     */
/* from several threads at once (one per device).                             */
/* ------------------------------------------------------------------------- */
typedef struct ks_engine_group ks_engine_group;

/* Number of visible CUDA devices. */
int32_t ks_device_count(void);
/* devices == NULL / n_devices <= 0: every visible device.  The same device may
 * appear more than once (several engines sharing a GPU). */
ks_status ks_engine_group_create_from_checkpoint(const char* path, const int32_t* devices, int32_t n_devices,
                                                 int32_t precision, ks_engine_group** out);
ks_status ks_engine_group_create(const ks_model_desc* model, const int32_t* devices, int32_t n_devices,
                                 int32_t precision, ks_engine_group** out);
void ks_engine_group_destroy(ks_engine_group* g);
int32_t ks_engine_group_size(const ks_engine_group* g);
ks_engine* ks_engine_group_engine(const ks_engine_group* g, int32_t i);
ks_status ks_group_beam_search_batch(ks_engine_group* g, const int32_t* tok, const int64_t* desc, int64_t B,
                                     int32_t beam_width, const ks_pred* preds, int32_t n_preds,
                                     ks_host_pred_fn hook, void* user, int32_t* out_tok, double* out_lp,
                                     int32_t* out_count, int32_t* out_status, int32_t* out_fail_pred,
                                     int32_t* out_fail_step);
ks_status ks_group_greedy_batch(ks_engine_group* g, const int32_t* tok, int64_t B, int32_t* out_tok);
ks_status ks_group_forward_batch(ks_engine_group* g, const int32_t* tok, const int32_t* teacher, int64_t B,
                                 double* out_dist, int32_t* out_tok, double* out_score);
/* Counters summed over the shards. */
ks_status ks_group_topk_metrics_multi(ks_engine_group* g, const int32_t* tok, const int64_t* desc,
                                      const int32_t* truth, int64_t B, const int32_t* k_values, int32_t n_k,
                                      const ks_pred* preds, int32_t n_preds, ks_host_pred_fn hook, void* user,
                                      int64_t* out_pos_matches, int64_t* out_perfect);
ks_status ks_group_topk_metrics_batch(ks_engine_group* g, const int32_t* tok, const int64_t* desc,
                                      const int32_t* truth, int64_t B, int32_t beam_width, const ks_pred* preds,
                                      int32_t n_preds, ks_host_pred_fn hook, void* user,
                                      int64_t* out_pos_matches, int64_t* out_perfect);

/* Kernel-level timing hook for bench.py: accumulated device milliseconds of
 * the gate-GEMM launches (CUDA events on the launching stream) since the last
 * reset, and their count. */
void ks_engine_profile_reset(ks_engine* eng, int32_t enable);
double ks_engine_profile_gemm_ms(const ks_engine* eng, int64_t* launches, double* useful_flops);
/* Per-launch view of the same profile: fills up to cap (ms, useful FLOPs)
 * pairs in launch order and returns the number of launches recorded. */
int64_t ks_engine_profile_launches(const ks_engine* eng, int64_t cap, double* ms, double* useful_flops);
/* Same, plus the FLOPs each launch issues to the tensor pipe (F16X3: three MMA
 * passes; the projected-context GEMMs contract fewer columns than the
 * reference's formula counts as useful). */
int64_t ks_engine_profile_launches_ex(const ks_engine* eng, int64_t cap, double* ms, double* useful_flops,
                                      double* mma_issued_flops);


/* ------------------------------------------------------------------------- */
/* Teacher-forced training (BASELINE config 4).  Replaces the batch body of   */
/* train_model (src/models.cpp:905-947: per-sample build_loss_graph +         */
/* Tape::backward, summed gradients, / batch, clip_global_norm, adam_step),   */
/* model_loss_gradients (src/models.cpp:788-797) summed over a batch, and     */
/* evaluate_set (src/models.cpp:827-856) for the enc-dec / attn / attn-2      */
/* variants.  fp32 parameters, moments and GEMMs; gradients are exchanged in  */
/* the "train layout" (ks_trainer_to_reference_layout converts).              */
/* ------------------------------------------------------------------------- */
typedef struct ks_trainer ks_trainer;

/* dropout / recurrent_dropout: ModelConfig::dropout / recurrent_dropout. */
ks_status ks_trainer_create(const ks_model_desc* model, double dropout, double recurrent_dropout,
                            int32_t device, ks_trainer** out);
/* dropout rates from the checkpoint header (data.cpp:478-479). */
ks_status ks_trainer_create_from_checkpoint(const char* path, int32_t device, ks_trainer** out);
void ks_trainer_destroy(ks_trainer* tr);
/* Length of the flat train-layout parameter / gradient buffers (segments padded
 * to 64 floats, so it is at least the reference parameter count). */
int64_t ks_trainer_num_params(const ks_trainer* tr);
/* The reference parameter count: length of the ks_trainer_export / import /
 * to_reference_layout host arrays. */
int64_t ks_trainer_num_ref_params(const ks_trainer* tr);
int64_t ks_trainer_last_launch_count(const ks_trainer* tr);

/* Forward + backward over B samples already on the device (d_tok B x 7 input
 * token ids, d_tgt B x T target token ids, d_idx B sample ids or NULL = 0..B-1).
 * dropout_epoch >= 0 with nonzero rates applies train_model's variational
 * dropout, each sample's masks drawn from Rng::derive(seed, epoch << 32 | idx)
 * (models.cpp:915-918); < 0 disables dropout (model_loss_gradients with a
 * null rng).  d_grads (num_params floats, train layout) receives the SUM over
 * the batch of the per-sample gradients (accumulate != 0 adds to it);
 * d_grads == NULL runs the forward only (evaluate_set).  d_loss_sum (1 double)
 * and d_matches (1 int64: per-position argmax hits) are device pointers, may
 * be NULL.  Asynchronous on `stream`. */
ks_status ks_trainer_loss_grads(ks_trainer* tr, const int32_t* d_tok, const int32_t* d_tgt,
                                const int64_t* d_idx, int64_t B, int64_t dropout_epoch,
                                uint64_t seed, float* d_grads, int32_t accumulate,
                                double* d_loss_sum, int64_t* d_matches, void* stream);
/* Optimiser step on summed gradients of `batch` samples (all ranks' sum after
 * an all-reduce): grads / batch, clip_global_norm(clip), adam_step(lr) with
 * AdamConfig defaults (nn.hpp:96-101).  Asynchronous on `stream`. */
ks_status ks_trainer_apply(ks_trainer* tr, const float* d_grads, int64_t batch, double lr, double clip,
                           void* stream);
/* Host-buffer single-GPU step (the reference-facing call): copies, loss_grads,
 * apply, and the loss sum / matches back to the host. */
ks_status ks_trainer_step(ks_trainer* tr, const int32_t* tok, const int32_t* tgt, const int64_t* idx,
                          int64_t B, int64_t epoch, uint64_t seed, double lr, double clip,
                          double* out_loss_sum, int64_t* out_matches);
/* Host-buffer forward only (evaluate_set, models.cpp:827-856): teacher-forced
 * loss sum and per-position argmax matches of B samples, dropout off. */
ks_status ks_trainer_evaluate(ks_trainer* tr, const int32_t* tok, const int32_t* tgt, int64_t B,
                              double* out_loss_sum, int64_t* out_matches);
/* Parameters in reference flat order (the model's tensors concatenated in
 * ks_model_desc / checkpoint order), to and from the host. */
ks_status ks_trainer_export(const ks_trainer* tr, float* host_ref_flat);
ks_status ks_trainer_import(ks_trainer* tr, const float* host_ref_flat);
/* Permutes a train-layout buffer (e.g. gradients) into reference flat order. */
ks_status ks_trainer_to_reference_layout(const ks_trainer* tr, const float* host_train_flat,
                                         float* host_ref_flat);

/* The training contractions' GEMM as a library call (csrc/ks_gemm16.cu), on
 * caller DEVICE buffers and stream: C[M x N] = op(A) op(B) + beta C, row-major
 * fp32; op(A) = A^T when ta (A stored K x M), op(B) = B^T when tb (B stored
 * N x K); beta 0 or 1.  F16X3 on tcgen05: both operands split into fp16 hi/lo
 * planes at power-of-two scales, hi.hi + hi.lo + lo.hi with fp32 accumulation
 * (fp32-grade; the reference's fp64 GEMMs are autodiff.cpp:326-544's matmuls).
 * Replaces the reference's training-time `matmul` (tensor.hpp / autodiff.cpp). */
ks_status ks_gemm_f16x3(int32_t ta, int32_t tb, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                        const float* B, int64_t ldb, float beta, float* C, int64_t ldc, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* KS_B200_H */
