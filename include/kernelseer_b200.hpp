// kernelseer_b200.hpp -- the reference's C++ hot-path API, served by the B200
// engine.  A caller of the reference library (kernelseer) that includes this
// header instead of kernelseer/{decoding,constraints,data,eval}.hpp and links
// libkernelseer_b200.so keeps its source unchanged for the decode path:
//
//   load_checkpoint            proj/include/kernelseer/data.hpp:77
//   SequencePredictor          proj/include/kernelseer/models.hpp:80-98 (facade; device engine inside)
//   greedy_decode, beam_search, constrained_beam_search
//                              proj/include/kernelseer/decoding.hpp:23-36
//   membership_predicate, resource_budget_predicate, ConstraintPredicate, validate_sequence
//                              proj/include/kernelseer/constraints.hpp:45-74
//   encode_problem, decode_params, encode_params, Vocabulary
//                              proj/include/kernelseer/encoding.hpp:17-95
//   topk_metrics, compute_metrics, EvalReport
//                              proj/include/kernelseer/eval.hpp:13-41
//   error classes              proj/include/kernelseer/errors.hpp:10-87
//
// Additions: batched entry points (beam_search_batch, greedy_decode_batch)
// and typed predicate factories for hardware limits (product_limit_predicate,
// divisibility_predicate).  Everything computes on the GPU through the C-ABI
// in ks_b200.h; opaque ConstraintPredicate::fn callables are evaluated on the
// host between positions by the engine's predicate hook.
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

struct ks_engine;
struct ks_engine_group;

namespace kernelseer {

// ---------------------------------------------------------------- errors
class Error : public std::runtime_error {
public:
    explicit Error(const std::string& m) : std::runtime_error(m) {}
};
class ShapeError : public Error { using Error::Error; };
class ParameterError : public Error { using Error::Error; };
class IndexError : public Error { using Error::Error; };
class StateError : public Error { using Error::Error; };
class ValidationError : public Error {
public:
    ValidationError(const std::string& m, std::string field) : Error(m), field_(std::move(field)) {}
    const std::string& field() const { return field_; }
private:
    std::string field_;
};
class CheckpointError : public Error {
public:
    enum class Kind { version, truncated, shape, malformed, io };
    CheckpointError(Kind k, const std::string& m) : Error(m), kind_(k) {}
    Kind kind() const { return kind_; }
private:
    Kind kind_;
};
class BeamExhaustedError : public Error {
public:
    BeamExhaustedError(const std::string& m, std::string predicate, int step)
        : Error(m), predicate_(std::move(predicate)), step_(step) {}
    const std::string& predicate() const { return predicate_; }
    int step() const { return step_; }
private:
    std::string predicate_;
    int step_;
};

// ---------------------------------------------------------------- tensors
namespace nn {
// The host fp64 tensor of the reference (tensor.hpp:13-55), reduced to what
// callers of the decode API touch: distributions returned by
// SequencePredictor::step / model_forward.
class Tensor {
public:
    Tensor() = default;
    explicit Tensor(std::vector<int> shape);
    Tensor(std::vector<int> shape, std::vector<double> data);
    static Tensor vec(std::vector<double> data);
    const std::vector<int>& shape() const { return shape_; }
    int rank() const { return static_cast<int>(shape_.size()); }
    int dim(int i) const { return shape_[static_cast<std::size_t>(i)]; }
    int size() const { return static_cast<int>(data_.size()); }
    bool empty() const { return data_.empty(); }
    double* data() { return data_.data(); }
    const double* data() const { return data_.data(); }
    std::vector<double>& values() { return data_; }
    const std::vector<double>& values() const { return data_; }
    double& operator[](int i) { return data_[static_cast<std::size_t>(i)]; }
    double operator[](int i) const { return data_[static_cast<std::size_t>(i)]; }
    double& at(int i, int j) { return data_[static_cast<std::size_t>(i) * shape_[1] + j]; }
    double at(int i, int j) const { return data_[static_cast<std::size_t>(i) * shape_[1] + j]; }

private:
    std::vector<int> shape_;
    std::vector<double> data_;
};
}  // namespace nn

// ---------------------------------------------------------------- problems
enum class Precision { full, half };
std::string precision_label(Precision p);
Precision precision_from_label(const std::string& s);

struct ProblemDescriptor {
    std::int64_t n = 1, c = 1, h_i = 1, w_i = 1, k = 1, y = 1, x = 1;
    Precision precision = Precision::full;
    bool operator==(const ProblemDescriptor&) const = default;
    void check() const;
};
inline constexpr int kNumInputFields = 7;
inline constexpr std::array<const char*, kNumInputFields> kInputFieldNames = {"n", "c", "h", "w",
                                                                            "k", "y", "x"};
std::int64_t descriptor_field(const ProblemDescriptor& d, int field);
void set_descriptor_field(ProblemDescriptor& d, int field, std::int64_t value);
using ParamMap = std::map<std::string, std::int64_t>;

// ---------------------------------------------------------------- kernel specs
struct KernelSpec {
    struct Param {
        std::string name;
        std::vector<std::int64_t> values;
    };
    std::string name;
    std::vector<Param> params;
    int num_params() const { return static_cast<int>(params.size()); }
    int param_index(std::string_view n) const;
    void check() const;
};
const std::vector<KernelSpec>& builtin_specs();
const KernelSpec& builtin_spec(std::string_view name);
std::uint64_t search_space_size(const KernelSpec& spec);

// ---------------------------------------------------------------- predicates
// Device form of a predicate (mirrors ks_pred): parameters are named, the
// engine resolves them against the model's output positions at call time.
struct PredicateProgram {
    enum class Kind { mask = 1, budget = 2, product = 3, divides = 4 };
    Kind kind = Kind::mask;
    // mask: legal values per parameter name (membership)
    std::map<std::string, std::vector<std::int64_t>> legal;
    // budget: weights by name (std::map -> alphabetical, as constraints.cpp:235)
    std::map<std::string, double> weights;
    double budget = 0.0;
    // product: scale * prod(values) <= limit
    std::vector<std::string> factors;
    std::int64_t scale = 1, limit = 0;
    // divides: (parameter, descriptor field index)
    std::vector<std::pair<std::string, int>> divides;
};

struct ConstraintPredicate {
    std::string name;
    std::vector<std::string> reads;
    bool full_sequence_only = false;
    std::function<bool(const ProblemDescriptor&, const ParamMap&)> fn;  // always set
    std::shared_ptr<const PredicateProgram> program;                     // typed factories only
    bool evaluate(const ProblemDescriptor& d, const ParamMap& m) const { return fn(d, m); }
};

ConstraintPredicate membership_predicate(const KernelSpec& spec);
ConstraintPredicate resource_budget_predicate(std::map<std::string, double> weights, double budget,
                                              std::string name = "resource_budget");
// New (no reference counterpart): workgroup size / LDS bytes style limits.
ConstraintPredicate product_limit_predicate(std::vector<std::string> params, std::int64_t scale,
                                            std::int64_t limit, std::string name = "product_limit");
// New: each listed parameter value must divide a descriptor field (0..6 = n,c,h,w,k,y,x).
ConstraintPredicate divisibility_predicate(std::vector<std::pair<std::string, int>> param_field,
                                           std::string name = "divisibility");

struct Violation {
    std::string predicate;
    std::vector<std::string> params;
};
std::optional<Violation> validate_sequence(const KernelSpec& spec, const ProblemDescriptor& d,
                                           const ParamMap& params,
                                           std::span<const ConstraintPredicate> predicates);

// ---------------------------------------------------------------- vocabulary
struct FieldVocab {
    std::string name;
    std::vector<std::int64_t> values;
    int size() const { return static_cast<int>(values.size()); }
    int id_of(std::int64_t v) const;
    std::int64_t value_of(int id) const;
    std::int64_t nearest(std::int64_t v) const;
};

class Vocabulary {
public:
    static constexpr int kGoToken = 0;
    Vocabulary() = default;
    Vocabulary(std::vector<FieldVocab> input_fields, std::vector<FieldVocab> output_params);
    const std::vector<FieldVocab>& input_fields() const { return in_; }
    const std::vector<FieldVocab>& output_params() const { return out_; }
    const FieldVocab& input_field(int i) const { return in_.at(static_cast<std::size_t>(i)); }
    const FieldVocab& output_param(int i) const { return out_.at(static_cast<std::size_t>(i)); }
    int num_output_positions() const { return static_cast<int>(out_.size()); }
private:
    std::vector<FieldVocab> in_, out_;
};

struct TokenSequence {
    enum class Role { input, output };
    Role role = Role::input;
    std::vector<int> ids;
    int length() const { return static_cast<int>(ids.size()); }
    bool operator==(const TokenSequence&) const = default;
};

TokenSequence encode_problem(const ProblemDescriptor& d, const Vocabulary& v, bool allow_nearest = false);
ProblemDescriptor decode_problem(const TokenSequence& t, const Vocabulary& v,
                                 Precision precision = Precision::full);
ParamMap decode_params(const TokenSequence& t, const KernelSpec& spec, const Vocabulary& v);
TokenSequence encode_params(const ParamMap& params, const KernelSpec& spec, const Vocabulary& v);

// ---------------------------------------------------------------- models
enum class ModelVariant { enc_dec, attn, attn2, hybrid, hybrid2 };
std::string variant_label(ModelVariant v);
ModelVariant variant_from_label(const std::string& s);

struct ConvLayerSpec {
    int filters = 64;
    int kernel_size = 3;
    int stride = 1;
};

struct ModelConfig {
    ModelVariant variant = ModelVariant::hybrid2;
    std::vector<ConvLayerSpec> conv_layers = {{64, 3, 1}, {32, 3, 1}};
    int encoder_state_size = 256;
    int pre_attention_size = 256;
    int post_attention_size = 512;
    int attention_dense_nodes = 2;
    int decoder_cell_size = 256;
    double dropout = 0.2;
    double recurrent_dropout = 0.2;
};

struct HostTensor {
    std::vector<int> shape;
    std::vector<float> values;  // checkpoints are fp32 (data.cpp:447-460)
};

struct ModelParams {
    ModelConfig config;
    std::string kernel;
    Precision precision = Precision::full;
    Vocabulary vocab;
    std::map<std::string, HostTensor> tensors;
    int num_output_positions() const { return vocab.num_output_positions(); }
};

KernelSpec spec_of(const ModelParams& params);
ModelParams load_checkpoint(const std::string& path);

// Benchmark / parity workloads (B200 addition, ks_synthetic_descriptors):
// configs start..start+count-1, config i drawn from Rng::derive(seed, i)
// uniformly with replacement over the model's input vocabulary.
std::vector<ProblemDescriptor> synthetic_descriptors(const ModelParams& params, std::int64_t count,
                                                     std::uint64_t seed = 2404, std::int64_t start = 0);

// GEMM arithmetic of the engine (see ks_b200.h).
enum class GemmPrecision { f16x3 = 0, fp32 = 1, bf16 = 2 };

// Per-input work shared by all hypotheses (models.hpp:65-70).  The encoder
// state lives on the device, so the host record keeps the input tokens; the
// reference's activations / h / c / dists members are kept for source
// compatibility and stay empty.
struct EncodedInput {
    TokenSequence input;
    std::vector<nn::Tensor> activations;
    nn::Tensor h, c;
    std::vector<nn::Tensor> dists;
};

// Per-hypothesis decoder state (models.hpp:72-76): the position and the tokens
// fed back so far (fed[q] = token emitted at position q); h / c are not
// materialised on the host.
struct DecoderState {
    nn::Tensor h, c;
    int position = 0;
    std::vector<int> fed;
};

// Stepping facade of the reference (models.hpp:78-98), here a handle on a
// device engine built from the params (weights packed and uploaded once,
// shared by copies).  Beam search does not go through step(): it runs whole
// batches on the device (beam_search_batch).  step() stays functional for API
// compatibility as a batch-of-1 device call (ks_forward_batch) that replays
// the decoder over the fed-back prefix: O(position) device work per call.
class SequencePredictor {
public:
    // device = kAllDevices: one engine per visible GPU, batches sharded across
    // them (the B200 counterpart of parallel_stripes over all host threads);
    // device >= 0: that GPU only.
    static constexpr int kAllDevices = -1;
    explicit SequencePredictor(const ModelParams& params, int device = kAllDevices,
                               GemmPrecision precision = GemmPrecision::f16x3);
    SequencePredictor(const ModelParams& params, std::vector<int> devices,
                      GemmPrecision precision = GemmPrecision::f16x3);
    int num_positions() const;
    int vocab_size(int position) const;
    const ModelParams& params() const { return *params_; }
    ks_engine* engine() const;           // the first device's engine
    ks_engine_group* group() const;      // every device's engine
    int num_devices() const;

    EncodedInput encode(const TokenSequence& input) const;
    DecoderState initial_state(const EncodedInput& enc) const;
    // Distribution for state.position; prev_token is the token emitted at the
    // previous position (ignored at position 0, which consumes GO).  Advances
    // the state; StateError past the last position, IndexError for a
    // prev_token outside the previous position's vocabulary.
    nn::Tensor step(const EncodedInput& enc, DecoderState& state, int prev_token) const;

private:
    void create(const std::vector<int>& devices, GemmPrecision precision);
    const ModelParams* params_;
    std::shared_ptr<ks_engine_group> group_;
};

// model_forward (models.hpp:100-103, models.cpp:495-514): per-position output
// distributions in infer mode; with teacher tokens the decoder consumes them
// as feedback, otherwise its own argmax.
std::vector<nn::Tensor> model_forward(const ModelParams& params, const TokenSequence& input,
                                      const std::vector<int>* teacher = nullptr);
// Same on an existing predictor's engine, and batched: one device pass over
// all inputs (teachers empty or one per input).  scores (optional) receives
// each input's sequence score sum_p log(max(p_p[token_p], 1e-300)).
std::vector<std::vector<nn::Tensor>> model_forward_batch(const SequencePredictor& predictor,
                                                         std::span<const TokenSequence> inputs,
                                                         std::span<const std::vector<int>> teachers = {},
                                                         std::vector<double>* scores = nullptr);

struct ScoredSequence {
    TokenSequence tokens;
    double log_prob = 0.0;
};

TokenSequence greedy_decode(const SequencePredictor& predictor, const TokenSequence& input);
std::vector<ScoredSequence> beam_search(const SequencePredictor& predictor, const TokenSequence& input,
                                        int beam_width);
std::vector<ScoredSequence> constrained_beam_search(const SequencePredictor& predictor,
                                                    const TokenSequence& input, int beam_width,
                                                    std::span<const ConstraintPredicate> predicates,
                                                    const ProblemDescriptor& descriptor);

// Batched forms (one device pass over all inputs).  Exhausted configs have an
// empty beam list and their BeamExhaustedError details in `exhausted`.
struct BatchResult {
    std::vector<std::vector<ScoredSequence>> beams;
    struct Exhaustion {
        bool exhausted = false;
        std::string predicate;
        int step = -1;
    };
    std::vector<Exhaustion> exhausted;
};
BatchResult beam_search_batch(const SequencePredictor& predictor, std::span<const TokenSequence> inputs,
                              std::span<const ProblemDescriptor> descriptors, int beam_width,
                              std::span<const ConstraintPredicate> predicates = {});
std::vector<TokenSequence> greedy_decode_batch(const SequencePredictor& predictor,
                                               std::span<const TokenSequence> inputs);

// ---------------------------------------------------------------- evaluation
struct Sample {
    ProblemDescriptor descriptor;
    ParamMap params;
    std::string kernel;
    Precision precision = Precision::full;
};

struct EvalReport {
    int beam_width = 1;
    bool constrained = false;
    int sample_count = 0;
    std::vector<double> per_param_accuracy;
    double average_accuracy = 0.0;
    double perfect_prediction = 0.0;
};

EvalReport compute_metrics(const std::vector<TokenSequence>& predictions,
                           const std::vector<TokenSequence>& actuals);
// `threads` is accepted for source compatibility; the batch runs on the GPU.
std::vector<EvalReport> topk_metrics(const ModelParams& params, const std::vector<Sample>& test,
                                     const std::vector<int>& k_values,
                                     std::span<const ConstraintPredicate> predicates = {},
                                     int threads = 1);
// Same, reusing an existing predictor's device engine.
std::vector<EvalReport> topk_metrics(const SequencePredictor& predictor, const std::vector<Sample>& test,
                                     const std::vector<int>& k_values,
                                     std::span<const ConstraintPredicate> predicates = {},
                                     int threads = 1);

// ------------------------------------------------------------------ training
// (models.hpp:139-169, data.hpp, rng.hpp).  The teacher-forced training loop
// of the reference, with each batch's forward / backward / Adam step on the
// GPU (ks_trainer_*, enc-dec / attn / attn-2).  Initialisation, the epoch
// shuffle and the per-sample dropout streams use the reference's Rng, so a
// run reproduces the reference's trajectory up to fp32 vs fp64 arithmetic.
class Rng {
public:
    explicit Rng(std::uint64_t seed);
    static Rng derive(std::uint64_t seed, std::uint64_t stream);
    std::uint64_t next_u64();
    double uniform();
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    std::uint64_t uniform_int(std::uint64_t n);

private:
    std::uint64_t mt_[312];
    int idx_ = 312;
};

struct TrainOptions {
    int epochs = 30;
    int batch_size = 32;
    std::uint64_t seed = 1;
    int threads = 1;          // accepted for source compatibility; batches run on the GPU
    double learning_rate = 1e-3;
    double clip_norm = 5.0;
};

struct EpochStats {
    int epoch = 0;
    double train_loss = 0.0;
    double train_accuracy = 0.0;  // per-position argmax accuracy, percent
    double test_loss = 0.0;
    double test_accuracy = 0.0;
};

struct TrainResult {
    ModelParams params;
    std::vector<EpochStats> log;
};

Vocabulary build_vocab(const KernelSpec& spec, const std::vector<Sample>& dataset);
ModelParams init_model(const ModelConfig& config, const KernelSpec& spec, const Vocabulary& vocab,
                       Precision precision, std::uint64_t seed);
TrainResult train_model(const ModelConfig& config, const KernelSpec& spec, const Vocabulary& vocab,
                        Precision precision, const std::vector<Sample>& train_set,
                        const std::vector<Sample>& test_set, const TrainOptions& options,
                        const std::function<void(const EpochStats&)>& on_epoch = {}, int device = 0);
void save_checkpoint(const ModelParams& params, const std::string& path);

}  // namespace kernelseer
