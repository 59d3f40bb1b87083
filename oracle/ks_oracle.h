/* ks_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, fp64 restatement of the reference's constrained-beam-decode hot
 * path (kernelseer, /root/reference/proj).  It is the CHECKER for the CUDA
 * product: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load it, and never as the thing measured or shipped.
 *
 * Arithmetic follows the reference operation by operation (same accumulation
 * order, separate multiply and add, glibc exp/log/tanh, compiled without FMA
 * contraction), so its results are bit-identical to the reference build; the
 * pinning tests (tests/test_oracle_pin.py) check exactly that against
 * oracle/_ref/libkernelseer_ref.so and the committed golden fixtures.
 */
#ifndef KS_ORACLE_H
#define KS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct kso_model kso_model;

/* load_checkpoint (proj/src/data.cpp:513-665): NULL on error, see kso_last_error. */
kso_model* kso_load(const char* path);
void kso_free(kso_model* m);
const char* kso_last_error(void);

/* variant: 0 enc-dec, 1 attn, 2 attn-2, 3 hybrid, 4 hybrid-2 (proj/include/kernelseer/models.hpp:16) */
int kso_variant(const kso_model* m);
int kso_num_positions(const kso_model* m);
int kso_vocab_size(const kso_model* m, int pos);
const char* kso_output_name(const kso_model* m, int pos);
int kso_input_vocab_size(const kso_model* m, int field);
int64_t kso_input_value(const kso_model* m, int field, int id);
int64_t kso_output_value(const kso_model* m, int pos, int id);
/* Mutable access to a named fp64 tensor (tests perturb weights); NULL if absent. */
double* kso_tensor(kso_model* m, const char* name, int* numel);

/* encode_problem (proj/src/encoding.cpp:87-113) without snapping: returns the
 * first field index whose value is out of vocabulary, or -1 when all 7 map. */
int kso_encode_problem(const kso_model* m, const int64_t* desc7, int32_t* tok7);

/* Typed predicate programs.  The reference's predicates are opaque
 * std::function objects (proj/include/kernelseer/constraints.hpp:45-54); the
 * product needs a device-evaluable form, and so does this checker. */
enum {
    KSO_PRED_MASK = 1,    /* allowed[value_offset(pos)+tok]; membership_predicate
                             (proj/src/constraints.cpp:198-218) and static masks */
    KSO_PRED_BUDGET = 2,  /* resource_budget_predicate (constraints.cpp:220-242):
                             sum over terms in ALPHABETICAL name order of w*value for
                             assigned params, separate mul/add in fp64, accept if <= budget */
    KSO_PRED_PRODUCT = 3, /* new (no reference counterpart): scale * prod(assigned values
                             of the listed positions) <= limit (workgroup / LDS bytes) */
    KSO_PRED_DIVIDES = 4  /* new: for each (pos, descriptor field) term with pos assigned:
                             value > 0 and desc[field] % value == 0 (tile divisibility) */
};

typedef struct {
    int kind;
    int full_sequence_only;      /* evaluated only at the last position (decoding.cpp:67-70) */
    const uint8_t* allowed;      /* MASK: sum_p V_p entries */
    int n_terms;                 /* BUDGET/PRODUCT/DIVIDES */
    const int32_t* term_pos;     /* output position of each term, -1 = never assigned */
    const double* term_w;        /* BUDGET weights (alphabetical order) */
    const int32_t* term_field;   /* DIVIDES: descriptor field 0..6 */
    double budget;               /* BUDGET */
    int64_t scale;               /* PRODUCT */
    int64_t limit;               /* PRODUCT */
} kso_pred;

/* beam_search_impl (proj/src/decoding.cpp:27-103).
 * Returns 0 on success, 1 when the constrained search exhausted (then
 * *fail_pred = index of the last rejecting predicate, *fail_step = position),
 * negative on argument errors.  out_tok: k*T, out_lp: k.
 * *min_gap receives the smallest relative log-prob gap between two candidates
 * whose order decided top-k membership (any position) or final rank. */
int kso_beam(const kso_model* m, const int32_t* tok7, const int64_t* desc7, int k,
             const kso_pred* preds, int n_preds, int32_t* out_tok, double* out_lp,
             int32_t* out_count, int32_t* fail_pred, int32_t* fail_step, double* min_gap);

/* greedy_decode (decoding.cpp:107-124): out_tok T entries. */
int kso_greedy(const kso_model* m, const int32_t* tok7, int32_t* out_tok);

/* model_forward (proj/src/models.cpp:495-514) with optional teacher tokens:
 * out: sum_p V_p probabilities. */
int kso_forward(const kso_model* m, const int32_t* tok7, const int32_t* teacher, double* out);

/* Encoder activations of the attention variants (models.cpp:401-408): out 7 x 2n_a. */
int kso_encode(const kso_model* m, const int32_t* tok7, double* out);

/* Batch helpers (loop over rows; threads <= 1 runs serially). */
int kso_beam_batch(const kso_model* m, const int32_t* tok, const int64_t* desc, int64_t B,
                   int k, const kso_pred* preds, int n_preds, int threads, int32_t* out_tok,
                   double* out_lp, int32_t* out_count, int32_t* out_status,
                   int32_t* out_fail_pred, int32_t* out_fail_step, double* out_min_gap);

/* ---- Rng (proj/include/kernelseer/rng.hpp:13-71): mt19937_64 + derive ---- */
/* Dropout masks of one sample as LstmMasks::make draws them
 * (proj/src/models.cpp:559-573, nn::dropout_mask nn.cpp:237-248) from the stream
 * Rng::derive(seed, stream): n_in input-mask entries (rate_in) then n_rec
 * recurrent-mask entries (rate_rec); out: n_in + n_rec values (0 or 1/(1-rate)). */
void kso_dropout_masks(uint64_t seed, uint64_t stream, int n_in, double rate_in, int n_rec,
                       double rate_rec, double* out);
/* train_model's per-epoch Fisher-Yates shuffle (proj/src/models.cpp:895-900):
 * order[0..n) from Rng::derive(seed, 0x3ff000 + epoch). */
void kso_shuffle(uint64_t seed, uint64_t epoch, int64_t n, int64_t* order);
/* Uniform draws of Rng::derive(seed, stream).uniform() (test hook). */
void kso_uniforms(uint64_t seed, uint64_t stream, int64_t n, double* out);

#ifdef __cplusplus
}
#endif
#endif
