// kernelseer_api.cpp -- the reference-compatible C++ host layer
// (include/kernelseer_b200.hpp) over the engine's C-ABI (include/ks_b200.h).
//
// Host-side work here is O(batch x positions) bookkeeping: descriptor
// tokenisation, predicate resolution, result unpacking, metrics.  All model
// arithmetic and the beam search run on the GPU.
#include "kernelseer_b200.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <sstream>

#include "ks_b200.h"

namespace kernelseer {

namespace {

[[noreturn]] void throw_status(ks_status st) {
    const std::string msg = ks_last_error();
    switch (st) {
        case KS_ERR_SHAPE: throw ShapeError(msg);
        case KS_ERR_PARAMETER: throw ParameterError(msg);
        case KS_ERR_INDEX: throw IndexError(msg);
        case KS_ERR_STATE: throw StateError(msg);
        case KS_ERR_VALIDATION: throw ValidationError(msg, ks_last_error_field());
        case KS_ERR_CHECKPOINT: {
            static const CheckpointError::Kind kinds[] = {
                CheckpointError::Kind::version, CheckpointError::Kind::truncated,
                CheckpointError::Kind::shape, CheckpointError::Kind::malformed,
                CheckpointError::Kind::io};
            const int k = ks_checkpoint_error_kind();
            throw CheckpointError(k >= 0 && k < 5 ? kinds[k] : CheckpointError::Kind::malformed, msg);
        }
        case KS_ERR_BEAM_EXHAUSTED: throw BeamExhaustedError(msg, "", -1);
        default: throw Error(msg);
    }
}

void check(ks_status st) {
    if (st != KS_OK) throw_status(st);
}

std::string join(const std::vector<std::int64_t>& v) {
    std::string s;
    for (std::size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + std::to_string(v[i]);
    return s;
}

}  // namespace

// ------------------------------------------------------------------ problems
std::string precision_label(Precision p) { return p == Precision::full ? "fp32" : "fp16"; }

Precision precision_from_label(const std::string& s) {
    if (s == "fp32" || s == "full") return Precision::full;
    if (s == "fp16" || s == "half") return Precision::half;
    throw ValidationError("unknown precision label '" + s + "' (expected fp32 or fp16)", "precision");
}

std::int64_t descriptor_field(const ProblemDescriptor& d, int f) {
    const std::int64_t v[7] = {d.n, d.c, d.h_i, d.w_i, d.k, d.y, d.x};
    if (f < 0 || f >= 7) throw IndexError("descriptor field index " + std::to_string(f));
    return v[f];
}

void set_descriptor_field(ProblemDescriptor& d, int f, std::int64_t value) {
    std::int64_t* v[7] = {&d.n, &d.c, &d.h_i, &d.w_i, &d.k, &d.y, &d.x};
    if (f < 0 || f >= 7) throw IndexError("descriptor field index " + std::to_string(f));
    *v[f] = value;
}

void ProblemDescriptor::check() const {
    for (int f = 0; f < kNumInputFields; ++f) {
        const std::int64_t v = descriptor_field(*this, f);
        if (v < 1)
            throw ValidationError(std::string("descriptor field ") + kInputFieldNames[f] +
                                      " must be >= 1, got " + std::to_string(v),
                                  kInputFieldNames[f]);
    }
}

// ------------------------------------------------------------------ kernel specs
int KernelSpec::param_index(std::string_view n) const {
    for (std::size_t i = 0; i < params.size(); ++i)
        if (params[i].name == n) return static_cast<int>(i);
    return -1;
}

void KernelSpec::check() const {
    if (params.empty()) throw ValidationError("kernel spec has no parameters", name);
    for (std::size_t i = 0; i < params.size(); ++i) {
        if (params[i].values.empty())
            throw ValidationError("parameter " + params[i].name + " has an empty value set", params[i].name);
        for (std::size_t j = 0; j < i; ++j)
            if (params[i].name == params[j].name)
                throw ValidationError("duplicate parameter name " + params[i].name, params[i].name);
    }
}

namespace {
std::vector<std::int64_t> span_of(std::int64_t lo, std::int64_t hi) {
    std::vector<std::int64_t> v;
    for (std::int64_t x = lo; x <= hi; ++x) v.push_back(x);
    return v;
}
std::vector<std::int64_t> pow2_of(int lo, int hi) {
    std::vector<std::int64_t> v;
    for (int e = lo; e <= hi; ++e) v.push_back(std::int64_t{1} << e);
    return v;
}
}  // namespace

// Table I of the paper (proj/tests/fixtures/table1.txt).
const std::vector<KernelSpec>& builtin_specs() {
    static const std::vector<KernelSpec> specs = [] {
        std::vector<KernelSpec> s;
        s.push_back({"ConvAsm1x1U",
                     {{"read_size", span_of(1, 4)}, {"k_mult", {1, 4, 8, 16, 32}},
                      {"chunks_per_wave", span_of(1, 16)}, {"chunk_size", pow2_of(0, 6)},
                      {"n_mult", span_of(1, 8)}, {"c_mult", pow2_of(0, 5)},
                      {"waves_c_in_group", span_of(1, 8)}, {"waves_k_in_group", pow2_of(0, 3)}}});
        s.push_back({"ConvOclDirectFwd1x1",
                     {{"grp_tile1", pow2_of(0, 4)}, {"grp_tile0", pow2_of(0, 8)}, {"in_tile1", pow2_of(0, 5)},
                      {"in_tile_0", pow2_of(0, 5)}, {"out_pix_tile1", {0, 1}}, {"out_pix_tile0", {0, 1, 2, 4}},
                      {"n_out_pix_tiles", pow2_of(0, 6)}, {"n_in_data_tiles", pow2_of(0, 11)},
                      {"n_stacks", {0, 1}}}});
        s.push_back({"ConvAsmBwdWrW1x1",
                     {{"read_size", span_of(1, 4)}, {"c_per_gpr", pow2_of(0, 4)}, {"c_mult", pow2_of(0, 4)},
                      {"k_per_gpr", pow2_of(0, 4)}, {"k_mult", pow2_of(0, 4)}, {"n_per_gpr", pow2_of(0, 4)},
                      {"n_part_cnt", span_of(1, 8)}, {"chunk_size", pow2_of(0, 4)}, {"short_store", {0, 1}},
                      {"data_prefetch", span_of(0, 4)}}});
        s.push_back({"ConvAsmBwdWrW3x3",
                     {{"limit_wave_cnt", span_of(0, 9)}, {"reverse_inout", {0, 1}}, {"chunk_size", {8, 16}},
                      {"k_per_wave", pow2_of(0, 3)}, {"pipe_lines_depth", span_of(1, 16)},
                      {"n_per_group", span_of(1, 8)}}});
        return s;
    }();
    return specs;
}

const KernelSpec& builtin_spec(std::string_view name) {
    std::string known;
    for (const KernelSpec& s : builtin_specs()) {
        if (s.name == name) return s;
        known += (known.empty() ? "" : ", ") + s.name;
    }
    throw ValidationError("unknown kernel '" + std::string(name) + "' (built-in: " + known + ")", "kernel");
}

std::uint64_t search_space_size(const KernelSpec& spec) {
    std::uint64_t n = 1;
    for (const auto& p : spec.params) n *= p.values.size();
    return n;
}

// ------------------------------------------------------------------ predicates
ConstraintPredicate membership_predicate(const KernelSpec& spec) {
    auto prog = std::make_shared<PredicateProgram>();
    prog->kind = PredicateProgram::Kind::mask;
    ConstraintPredicate p;
    p.name = "membership:" + spec.name;
    for (const auto& q : spec.params) {
        p.reads.push_back(q.name);
        prog->legal[q.name] = q.values;
    }
    p.program = prog;
    p.fn = [spec](const ProblemDescriptor&, const ParamMap& assigned) {
        for (const auto& [name, value] : assigned) {
            const int i = spec.param_index(name);
            if (i < 0)
                throw ValidationError("membership predicate: unknown parameter '" + name + "' for kernel " +
                                          spec.name,
                                      name);
            const auto& vals = spec.params[static_cast<std::size_t>(i)].values;
            if (std::find(vals.begin(), vals.end(), value) == vals.end()) return false;
        }
        return true;
    };
    return p;
}

ConstraintPredicate resource_budget_predicate(std::map<std::string, double> weights, double budget,
                                              std::string name) {
    for (const auto& [n, w] : weights)
        if (w < 0.0)
            throw ParameterError("resource budget weight for " + n + " must be nonnegative, got " +
                                 std::to_string(w));
    if (budget < 0.0) throw ParameterError("resource budget must be nonnegative");
    auto prog = std::make_shared<PredicateProgram>();
    prog->kind = PredicateProgram::Kind::budget;
    prog->weights = weights;
    prog->budget = budget;
    ConstraintPredicate p;
    p.name = std::move(name);
    for (const auto& [n, w] : weights) p.reads.push_back(n);
    p.program = prog;
    p.fn = [weights, budget](const ProblemDescriptor&, const ParamMap& assigned) {
        double cost = 0.0;  // alphabetical (std::map) order, separate multiply and add
        for (const auto& [n, w] : weights) {
            auto it = assigned.find(n);
            if (it == assigned.end()) continue;
            const volatile double prod = w * static_cast<double>(it->second);
            cost = cost + prod;
        }
        return cost <= budget;
    };
    return p;
}

ConstraintPredicate product_limit_predicate(std::vector<std::string> params, std::int64_t scale,
                                            std::int64_t limit, std::string name) {
    auto prog = std::make_shared<PredicateProgram>();
    prog->kind = PredicateProgram::Kind::product;
    prog->factors = params;
    prog->scale = scale;
    prog->limit = limit;
    ConstraintPredicate p;
    p.name = std::move(name);
    p.reads = params;
    p.program = prog;
    p.fn = [params, scale, limit](const ProblemDescriptor&, const ParamMap& assigned) {
        const __int128 cap = (__int128)1 << 100;
        __int128 prod = scale;
        for (const auto& n : params) {
            auto it = assigned.find(n);
            if (it == assigned.end()) continue;
            prod *= (__int128)it->second;
            prod = std::clamp(prod, -cap, cap);
        }
        return prod <= (__int128)limit;
    };
    return p;
}

ConstraintPredicate divisibility_predicate(std::vector<std::pair<std::string, int>> param_field,
                                           std::string name) {
    for (const auto& pf : param_field)
        if (pf.second < 0 || pf.second > 6) throw IndexError("descriptor field index " + std::to_string(pf.second));
    auto prog = std::make_shared<PredicateProgram>();
    prog->kind = PredicateProgram::Kind::divides;
    prog->divides = param_field;
    ConstraintPredicate p;
    p.name = std::move(name);
    for (const auto& pf : param_field) p.reads.push_back(pf.first);
    p.program = prog;
    p.fn = [param_field](const ProblemDescriptor& d, const ParamMap& assigned) {
        for (const auto& [n, f] : param_field) {
            auto it = assigned.find(n);
            if (it == assigned.end()) continue;
            if (it->second <= 0 || descriptor_field(d, f) % it->second != 0) return false;
        }
        return true;
    };
    return p;
}

std::optional<Violation> validate_sequence(const KernelSpec& spec, const ProblemDescriptor& d,
                                           const ParamMap& params,
                                           std::span<const ConstraintPredicate> predicates) {
    if (static_cast<int>(params.size()) != spec.num_params())
        throw ParameterError("validate_sequence: map has " + std::to_string(params.size()) + " entries, kernel " +
                             spec.name + " has " + std::to_string(spec.num_params()) + " parameters");
    for (const auto& p : spec.params)
        if (!params.contains(p.name)) throw ParameterError("validate_sequence: map missing parameter " + p.name);
    for (const auto& pred : predicates)
        if (!pred.evaluate(d, params)) return Violation{pred.name, pred.reads};
    return std::nullopt;
}

// ------------------------------------------------------------------ vocabulary
int FieldVocab::id_of(std::int64_t v) const {
    for (std::size_t i = 0; i < values.size(); ++i)
        if (values[i] == v) return static_cast<int>(i);
    return -1;
}

std::int64_t FieldVocab::value_of(int id) const {
    if (id < 0 || id >= size())
        throw IndexError("token id " + std::to_string(id) + " out of range for " + name + " (size " +
                         std::to_string(size()) + ")");
    return values[static_cast<std::size_t>(id)];
}

std::int64_t FieldVocab::nearest(std::int64_t v) const {
    std::int64_t best = values.front();
    for (std::int64_t x : values) {
        const std::int64_t dx = x > v ? x - v : v - x, db = best > v ? best - v : v - best;
        if (dx < db || (dx == db && x < best)) best = x;
    }
    return best;
}

Vocabulary::Vocabulary(std::vector<FieldVocab> in, std::vector<FieldVocab> out)
    : in_(std::move(in)), out_(std::move(out)) {}

TokenSequence encode_problem(const ProblemDescriptor& d, const Vocabulary& v, bool allow_nearest) {
    d.check();
    TokenSequence t;
    t.role = TokenSequence::Role::input;
    for (int f = 0; f < kNumInputFields; ++f) {
        const FieldVocab& fv = v.input_field(f);
        std::int64_t value = descriptor_field(d, f);
        int id = fv.id_of(value);
        if (id < 0 && allow_nearest) id = fv.id_of(fv.nearest(value));
        if (id < 0)
            throw ValidationError("value " + std::to_string(value) + " of field " + fv.name +
                                      " is not in the vocabulary (nearest known: " +
                                      std::to_string(fv.nearest(value)) + ")",
                                  fv.name);
        t.ids.push_back(id);
    }
    return t;
}

ProblemDescriptor decode_problem(const TokenSequence& t, const Vocabulary& v, Precision precision) {
    if (t.length() != kNumInputFields)
        throw ParameterError("decode_problem: expected 7 tokens, got " + std::to_string(t.length()));
    ProblemDescriptor d;
    d.precision = precision;
    for (int f = 0; f < kNumInputFields; ++f) set_descriptor_field(d, f, v.input_field(f).value_of(t.ids[f]));
    return d;
}

ParamMap decode_params(const TokenSequence& t, const KernelSpec& spec, const Vocabulary& v) {
    if (t.length() != spec.num_params())
        throw ParameterError("decode_params: sequence length " + std::to_string(t.length()) + " vs " +
                             std::to_string(spec.num_params()) + " parameters of " + spec.name);
    ParamMap out;
    for (int i = 0; i < spec.num_params(); ++i)
        out[spec.params[static_cast<std::size_t>(i)].name] = v.output_param(i).value_of(t.ids[static_cast<std::size_t>(i)]);
    return out;
}

TokenSequence encode_params(const ParamMap& params, const KernelSpec& spec, const Vocabulary& v) {
    if (static_cast<int>(params.size()) != spec.num_params())
        throw ParameterError("encode_params: map size " + std::to_string(params.size()) + " vs " +
                             std::to_string(spec.num_params()) + " parameters of " + spec.name);
    TokenSequence t;
    t.role = TokenSequence::Role::output;
    for (int i = 0; i < spec.num_params(); ++i) {
        const std::string& n = spec.params[static_cast<std::size_t>(i)].name;
        auto it = params.find(n);
        if (it == params.end()) throw ValidationError("encode_params: map missing parameter " + n, n);
        const int id = v.output_param(i).id_of(it->second);
        if (id < 0)
            throw ValidationError("value " + std::to_string(it->second) + " of parameter " + n +
                                      " is not in the vocabulary",
                                  n);
        t.ids.push_back(id);
    }
    return t;
}

// ------------------------------------------------------------------ models
std::string variant_label(ModelVariant v) {
    switch (v) {
        case ModelVariant::enc_dec: return "enc-dec";
        case ModelVariant::attn: return "attn";
        case ModelVariant::attn2: return "attn-2";
        case ModelVariant::hybrid: return "hybrid";
        case ModelVariant::hybrid2: return "hybrid-2";
    }
    throw ParameterError("unknown model variant");
}

ModelVariant variant_from_label(const std::string& s) {
    if (s == "enc-dec") return ModelVariant::enc_dec;
    if (s == "attn") return ModelVariant::attn;
    if (s == "attn-2") return ModelVariant::attn2;
    if (s == "hybrid") return ModelVariant::hybrid;
    if (s == "hybrid-2") return ModelVariant::hybrid2;
    throw ValidationError("unknown model variant '" + s + "' (enc-dec|attn|attn-2|hybrid|hybrid-2)", "variant");
}

KernelSpec spec_of(const ModelParams& params) {
    KernelSpec s;
    s.name = params.kernel;
    for (const FieldVocab& fv : params.vocab.output_params()) s.params.push_back({fv.name, fv.values});
    s.check();
    return s;
}

ModelParams load_checkpoint(const std::string& path) {
    ks_checkpoint* ck = nullptr;
    check(ks_checkpoint_load(path.c_str(), &ck));
    std::unique_ptr<ks_checkpoint, void (*)(ks_checkpoint*)> guard(ck, ks_checkpoint_free);
    auto hdr = [&](const char* k) -> std::string {
        const char* v = ks_checkpoint_header(ck, k);
        return v ? std::string(v) : std::string();
    };
    auto ints = [](const std::string& s) {
        std::vector<std::int64_t> v;
        std::stringstream ss(s);
        std::string piece;
        while (std::getline(ss, piece, ','))
            if (!piece.empty()) v.push_back(std::stoll(piece));
        return v;
    };
    ModelParams mp;
    mp.config.variant = variant_from_label(hdr("variant"));
    mp.kernel = hdr("kernel");
    if (!hdr("precision").empty()) mp.precision = precision_from_label(hdr("precision"));
    auto geti = [&](const char* k, int& dst) {
        const std::string v = hdr(k);
        if (!v.empty()) dst = std::stoi(v);
    };
    geti("encoder_state_size", mp.config.encoder_state_size);
    geti("pre_attention_size", mp.config.pre_attention_size);
    geti("post_attention_size", mp.config.post_attention_size);
    geti("attention_dense_nodes", mp.config.attention_dense_nodes);
    geti("decoder_cell_size", mp.config.decoder_cell_size);
    if (!hdr("conv_layers").empty()) {
        mp.config.conv_layers.clear();
        std::stringstream ss(hdr("conv_layers"));
        std::string layer;
        while (std::getline(ss, layer, ';')) {
            const auto v = ints(layer);
            if (v.size() != 3) throw CheckpointError(CheckpointError::Kind::malformed, "bad conv layer spec: " + layer);
            mp.config.conv_layers.push_back({(int)v[0], (int)v[1], (int)v[2]});
        }
    }
    if (!hdr("dropout").empty()) mp.config.dropout = std::stod(hdr("dropout"));
    if (!hdr("recurrent_dropout").empty()) mp.config.recurrent_dropout = std::stod(hdr("recurrent_dropout"));
    std::vector<FieldVocab> in, out;
    for (int f = 0; f < kNumInputFields; ++f) {
        const std::string v = hdr((std::string("input_vocab.") + kInputFieldNames[f]).c_str());
        if (v.empty())
            throw CheckpointError(CheckpointError::Kind::malformed,
                                  std::string("missing input vocabulary for field ") + kInputFieldNames[f]);
        in.push_back({kInputFieldNames[f], ints(v)});
    }
    const int np = hdr("output_params").empty() ? 0 : std::stoi(hdr("output_params"));
    for (int i = 0; i < np; ++i) {
        const std::string v = hdr(("param." + std::to_string(i)).c_str());
        const auto eq = v.find(" = ");
        if (eq == std::string::npos)
            throw CheckpointError(CheckpointError::Kind::malformed, "bad param header line: param." + std::to_string(i));
        out.push_back({v.substr(0, eq), ints(v.substr(eq + 3))});
    }
    mp.vocab = Vocabulary(std::move(in), std::move(out));
    for (int i = 0; i < ks_checkpoint_num_tensors(ck); ++i) {
        const char* name;
        int32_t rank = 0, dims[3] = {1, 1, 1};
        const float* data;
        check(ks_checkpoint_tensor(ck, i, &name, &rank, dims, &data));
        HostTensor t;
        std::size_t n = 1;
        for (int r = 0; r < rank; ++r) {
            t.shape.push_back(dims[r]);
            n *= static_cast<std::size_t>(dims[r]);
        }
        t.values.assign(data, data + n);
        mp.tensors.emplace(name, std::move(t));
    }
    return mp;
}

// ------------------------------------------------------------------ predictor
SequencePredictor::SequencePredictor(const ModelParams& params, int device, GemmPrecision precision)
    : params_(&params) {
    create(device == kAllDevices ? std::vector<int>{} : std::vector<int>{device}, precision);
}

SequencePredictor::SequencePredictor(const ModelParams& params, std::vector<int> devices, GemmPrecision precision)
    : params_(&params) {
    if (devices.empty()) throw ParameterError("empty device list");
    create(devices, precision);
}

void SequencePredictor::create(const std::vector<int>& devices, GemmPrecision precision) {
    const ModelParams& params = *params_;
    const int var = static_cast<int>(params.config.variant);
    std::vector<int32_t> in_sizes, vsizes;
    std::vector<int64_t> in_vals, out_vals;
    for (const auto& f : params.vocab.input_fields()) {
        in_sizes.push_back(f.size());
        in_vals.insert(in_vals.end(), f.values.begin(), f.values.end());
    }
    for (const auto& f : params.vocab.output_params()) {
        vsizes.push_back(f.size());
        out_vals.insert(out_vals.end(), f.values.begin(), f.values.end());
    }
    std::vector<const char*> names;
    std::vector<int32_t> numel;
    std::vector<const float*> data;
    for (const auto& [n, t] : params.tensors) {
        names.push_back(n.c_str());
        numel.push_back(static_cast<int32_t>(t.values.size()));
        data.push_back(t.values.data());
    }
    std::vector<int32_t> conv;
    for (const auto& l : params.config.conv_layers) {
        conv.push_back(l.filters);
        conv.push_back(l.kernel_size);
        conv.push_back(l.stride);
    }
    ks_model_desc d{};
    d.variant = var;
    d.decoder_cell_size = params.config.decoder_cell_size;
    d.num_conv_layers = static_cast<int32_t>(params.config.conv_layers.size());
    d.conv_layers = conv.data();
    d.encoder_state_size = params.config.encoder_state_size;
    d.pre_attention_size = params.config.pre_attention_size;
    d.post_attention_size = params.config.post_attention_size;
    d.attention_dense_nodes = params.config.attention_dense_nodes;
    d.num_positions = params.num_output_positions();
    d.input_sizes = in_sizes.data();
    d.input_values = in_vals.data();
    d.vocab_sizes = vsizes.data();
    d.output_values = out_vals.data();
    d.num_tensors = static_cast<int32_t>(names.size());
    d.tensor_names = names.data();
    d.tensor_numel = numel.data();
    d.tensor_data = data.data();
    ks_engine_group* g = nullptr;
    check(ks_engine_group_create(&d, devices.empty() ? nullptr : devices.data(), static_cast<int32_t>(devices.size()),
                                 static_cast<int32_t>(precision), &g));
    group_ = std::shared_ptr<ks_engine_group>(g, ks_engine_group_destroy);
}

int SequencePredictor::num_positions() const { return params_->num_output_positions(); }
int SequencePredictor::vocab_size(int position) const { return params_->vocab.output_param(position).size(); }
ks_engine* SequencePredictor::engine() const { return ks_engine_group_engine(group_.get(), 0); }
ks_engine_group* SequencePredictor::group() const { return group_.get(); }
int SequencePredictor::num_devices() const { return ks_engine_group_size(group_.get()); }

// ------------------------------------------------------------------ nn::Tensor
namespace nn {
Tensor::Tensor(std::vector<int> shape) : shape_(std::move(shape)) {
    std::size_t n = 1;
    for (int d : shape_) {
        if (d < 0) throw ShapeError("negative tensor dimension");
        n *= static_cast<std::size_t>(d);
    }
    data_.assign(n, 0.0);
}
Tensor::Tensor(std::vector<int> shape, std::vector<double> data) : shape_(std::move(shape)), data_(std::move(data)) {
    std::size_t n = 1;
    for (int d : shape_) n *= static_cast<std::size_t>(d);
    if (n != data_.size()) throw ShapeError("tensor data size does not match its shape");
}
Tensor Tensor::vec(std::vector<double> data) {
    const int n = static_cast<int>(data.size());
    return Tensor({n}, std::move(data));
}
}  // namespace nn

// ------------------------------------------------------------------ stepping facade
std::vector<std::vector<nn::Tensor>> model_forward_batch(const SequencePredictor& predictor,
                                                         std::span<const TokenSequence> inputs,
                                                         std::span<const std::vector<int>> teachers,
                                                         std::vector<double>* scores) {
    const int T = predictor.num_positions();
    const std::size_t B = inputs.size();
    if (!teachers.empty() && teachers.size() != B)
        throw ParameterError("model_forward_batch: " + std::to_string(teachers.size()) + " teachers for " +
                             std::to_string(B) + " inputs");
    std::vector<int32_t> tok(B * 7), tch(teachers.empty() ? 0 : B * T);
    for (std::size_t b = 0; b < B; ++b) {
        if (inputs[b].length() != kNumInputFields)
            throw ParameterError("model input must have 7 tokens, got " + std::to_string(inputs[b].length()));
        for (int f = 0; f < 7; ++f) tok[b * 7 + f] = inputs[b].ids[static_cast<std::size_t>(f)];
        if (!teachers.empty()) {
            if (static_cast<int>(teachers[b].size()) != T)  // models.cpp:499-503
                throw ParameterError("teacher sequence length " + std::to_string(teachers[b].size()) + " vs " +
                                     std::to_string(T) + " output positions");
            for (int p = 0; p < T; ++p) tch[b * T + p] = teachers[b][static_cast<std::size_t>(p)];
        }
    }
    std::vector<int> off(T + 1, 0);
    for (int p = 0; p < T; ++p) off[p + 1] = off[p] + predictor.vocab_size(p);
    std::vector<double> dist(B * off[T]), sc(B);
    if (B)
        check(ks_group_forward_batch(predictor.group(), tok.data(), tch.empty() ? nullptr : tch.data(),
                               static_cast<int64_t>(B), dist.data(), nullptr, sc.data()));
    std::vector<std::vector<nn::Tensor>> out(B);
    for (std::size_t b = 0; b < B; ++b)
        for (int p = 0; p < T; ++p)
            out[b].push_back(nn::Tensor::vec(std::vector<double>(dist.begin() + b * off[T] + off[p],
                                                                 dist.begin() + b * off[T] + off[p + 1])));
    if (scores) *scores = std::move(sc);
    return out;
}

std::vector<nn::Tensor> model_forward(const ModelParams& params, const TokenSequence& input,
                                      const std::vector<int>* teacher) {
    const SequencePredictor predictor(params);
    std::vector<std::vector<int>> t;
    if (teacher) t.push_back(*teacher);
    return model_forward_batch(predictor, std::span<const TokenSequence>(&input, 1),
                               std::span<const std::vector<int>>(t))[0];
}

EncodedInput SequencePredictor::encode(const TokenSequence& input) const {
    if (input.length() != kNumInputFields)  // models.cpp:112-116
        throw ParameterError("model input must have 7 tokens, got " + std::to_string(input.length()));
    for (int f = 0; f < kNumInputFields; ++f) {
        const int t = input.ids[static_cast<std::size_t>(f)];
        if (t < 0 || t >= params_->vocab.input_field(f).size())  // input_onehot, encoding.cpp:182-190
            throw IndexError("input_onehot: token " + std::to_string(t) + " out of range for field " +
                             params_->vocab.input_field(f).name);
    }
    EncodedInput enc;
    enc.input = input;
    return enc;
}

DecoderState SequencePredictor::initial_state(const EncodedInput&) const { return DecoderState{}; }

nn::Tensor SequencePredictor::step(const EncodedInput& enc, DecoderState& state, int prev_token) const {
    const int T = num_positions();
    const int pos = state.position;
    if (pos < 0 || pos >= T) throw StateError("decoder stepped past the last output position");  // models.cpp:452-454
    if (static_cast<int>(state.fed.size()) != std::max(0, pos - 1))
        throw StateError("decoder state does not match its position");
    const ModelVariant var = params_->config.variant;
    const bool feedback = var == ModelVariant::attn || var == ModelVariant::enc_dec;
    if (pos > 0) {
        if (feedback && (prev_token < 0 || prev_token >= vocab_size(pos - 1)))  // encoding.cpp:192-199
            throw IndexError("feedback_onehot: token " + std::to_string(prev_token) + " out of range for position " +
                             std::to_string(pos - 1));
        state.fed.push_back(feedback ? prev_token : 0);
    }
    std::vector<int> teacher(static_cast<std::size_t>(T), 0);
    std::copy(state.fed.begin(), state.fed.end(), teacher.begin());
    const std::vector<int> one[1] = {teacher};
    auto d = model_forward_batch(*this, std::span<const TokenSequence>(&enc.input, 1),
                                 std::span<const std::vector<int>>(one, 1));
    state.position = pos + 1;
    return std::move(d[0][static_cast<std::size_t>(pos)]);
}

std::vector<ProblemDescriptor> synthetic_descriptors(const ModelParams& params, std::int64_t count,
                                                     std::uint64_t seed, std::int64_t start) {
    if (count < 0 || start < 0) throw ParameterError("synthetic_descriptors: negative count / start");
    std::vector<int32_t> sizes;
    std::vector<int64_t> vals;
    for (const auto& f : params.vocab.input_fields()) {
        sizes.push_back(f.size());
        vals.insert(vals.end(), f.values.begin(), f.values.end());
    }
    if (sizes.size() != kNumInputFields) throw StateError("model has no input vocabulary");
    std::vector<int64_t> raw(static_cast<std::size_t>(count) * 7);
    check(ks_synthetic_descriptors(sizes.data(), vals.data(), seed, start, count, raw.data()));
    std::vector<ProblemDescriptor> out(static_cast<std::size_t>(count));
    for (std::int64_t i = 0; i < count; ++i)
        for (int f = 0; f < 7; ++f) set_descriptor_field(out[static_cast<std::size_t>(i)], f, raw[i * 7 + f]);
    return out;
}

// ------------------------------------------------------------------ decode
namespace {

// Resolved predicate list for one model: ks_pred array + backing storage + the
// opaque (host) predicates.
struct ResolvedPreds {
    std::vector<ks_pred> preds;
    std::vector<std::vector<uint8_t>> masks;
    std::vector<std::vector<int32_t>> pos, field;
    std::vector<std::vector<double>> w;
    std::vector<int> host;  // registration indices of opaque predicates
};

ResolvedPreds resolve(const ModelParams& mp, std::span<const ConstraintPredicate> preds) {
    ResolvedPreds r;
    const auto& outs = mp.vocab.output_params();
    auto pos_of = [&](const std::string& n) {
        for (std::size_t i = 0; i < outs.size(); ++i)
            if (outs[i].name == n) return static_cast<int32_t>(i);
        return -1;
    };
    r.preds.resize(preds.size());
    r.masks.resize(preds.size());
    r.pos.resize(preds.size());
    r.field.resize(preds.size());
    r.w.resize(preds.size());
    for (std::size_t i = 0; i < preds.size(); ++i) {
        const ConstraintPredicate& p = preds[i];
        ks_pred& q = r.preds[i];
        std::memset(&q, 0, sizeof q);
        q.full_sequence_only = p.full_sequence_only ? 1 : 0;
        if (!p.program) {
            q.kind = KS_PRED_HOST;
            r.host.push_back(static_cast<int>(i));
            continue;
        }
        const PredicateProgram& g = *p.program;
        switch (g.kind) {
            case PredicateProgram::Kind::mask: {
                q.kind = KS_PRED_MASK;
                for (const auto& f : outs) {
                    auto it = g.legal.find(f.name);
                    if (it == g.legal.end())
                        throw ValidationError("membership predicate: unknown parameter '" + f.name + "'", f.name);
                    for (std::int64_t v : f.values)
                        r.masks[i].push_back(std::find(it->second.begin(), it->second.end(), v) != it->second.end());
                }
                q.allowed = r.masks[i].data();
                break;
            }
            case PredicateProgram::Kind::budget:
                q.kind = KS_PRED_BUDGET;
                for (const auto& [n, w] : g.weights) {  // std::map: alphabetical
                    r.pos[i].push_back(pos_of(n));
                    r.w[i].push_back(w);
                }
                q.n_terms = static_cast<int32_t>(r.pos[i].size());
                q.term_pos = r.pos[i].data();
                q.term_w = r.w[i].data();
                q.budget = g.budget;
                break;
            case PredicateProgram::Kind::product:
                q.kind = KS_PRED_PRODUCT;
                for (const auto& n : g.factors) r.pos[i].push_back(pos_of(n));
                q.n_terms = static_cast<int32_t>(r.pos[i].size());
                q.term_pos = r.pos[i].data();
                q.scale = g.scale;
                q.limit = g.limit;
                break;
            case PredicateProgram::Kind::divides:
                q.kind = KS_PRED_DIVIDES;
                for (const auto& [n, f] : g.divides) {
                    r.pos[i].push_back(pos_of(n));
                    r.field[i].push_back(f);
                }
                q.n_terms = static_cast<int32_t>(r.pos[i].size());
                q.term_pos = r.pos[i].data();
                q.term_field = r.field[i].data();
                break;
        }
    }
    return r;
}

// The hook runs on one host thread per device of the predictor's group; the
// predicates themselves are called concurrently, as the reference calls them
// from its parallel_stripes workers.
struct HookCtx {
    const ModelParams* mp;
    std::span<const ConstraintPredicate> preds;
    const std::vector<int>* host;
    std::span<const ProblemDescriptor> descs;
    std::string error;
    std::mutex mu;  // guards error
};

// Evaluates the opaque predicates exactly as beam_search_impl does
// (decoding.cpp:60-77): decoded-value ParamMap of the child's prefix,
// registration order, full_sequence_only only at the last position.
int32_t host_hook(void* user, int32_t position, int32_t final_step, int64_t n_rows, const int32_t* row_config,
                  const int32_t* row_prefix, int32_t vocab, int32_t* out) {
    auto* ctx = static_cast<HookCtx*>(user);
    const auto& outs = ctx->mp->vocab.output_params();
    try {
        for (int64_t r = 0; r < n_rows; ++r) {
            ParamMap m;
            for (int t = 0; t < position; ++t)
                m[outs[static_cast<std::size_t>(t)].name] =
                    outs[static_cast<std::size_t>(t)].value_of(row_prefix[r * position + t]);
            const ProblemDescriptor& d = ctx->descs[static_cast<std::size_t>(row_config[r])];
            const std::string& name = outs[static_cast<std::size_t>(position)].name;
            for (int v = 0; v < vocab; ++v) {
                m[name] = outs[static_cast<std::size_t>(position)].value_of(v);
                int32_t rej = -1;
                for (int qi : *ctx->host) {
                    const ConstraintPredicate& q = ctx->preds[static_cast<std::size_t>(qi)];
                    if (q.full_sequence_only && !final_step) continue;
                    if (!q.evaluate(d, m)) {
                        rej = qi;
                        break;
                    }
                }
                out[r * vocab + v] = rej;
            }
        }
    } catch (const std::exception& e) {
        std::lock_guard<std::mutex> g(ctx->mu);
        if (ctx->error.empty()) ctx->error = e.what();
        return 1;
    }
    return 0;
}

}  // namespace

BatchResult beam_search_batch(const SequencePredictor& predictor, std::span<const TokenSequence> inputs,
                              std::span<const ProblemDescriptor> descriptors, int beam_width,
                              std::span<const ConstraintPredicate> predicates) {
    if (beam_width < 1) throw ParameterError("beam width must be >= 1, got " + std::to_string(beam_width));
    const ModelParams& mp = predictor.params();
    const int T = mp.num_output_positions();
    const std::size_t B = inputs.size();
    std::vector<int32_t> tok(B * 7);
    for (std::size_t b = 0; b < B; ++b) {
        if (inputs[b].length() != kNumInputFields)
            throw ParameterError("model input must have 7 tokens, got " + std::to_string(inputs[b].length()));
        for (int f = 0; f < 7; ++f) tok[b * 7 + f] = inputs[b].ids[static_cast<std::size_t>(f)];
    }
    std::vector<int64_t> desc;
    if (!descriptors.empty()) {
        if (descriptors.size() != B) throw ParameterError("descriptor count differs from input count");
        desc.resize(B * 7);
        for (std::size_t b = 0; b < B; ++b)
            for (int f = 0; f < 7; ++f) desc[b * 7 + f] = descriptor_field(descriptors[b], f);
    }
    ResolvedPreds rp = resolve(mp, predicates);
    if (!rp.host.empty() && descriptors.empty())
        throw ParameterError("opaque predicates need the problem descriptors");
    const std::size_t k = static_cast<std::size_t>(beam_width);
    std::vector<int32_t> otok(B * k * T), cnt(B), st(B), fp(B), fs(B);
    std::vector<double> olp(B * k);
    HookCtx ctx{&mp, predicates, &rp.host, descriptors, {}};
    ks_status s = ks_group_beam_search_batch(
        predictor.group(), tok.data(), desc.empty() ? nullptr : desc.data(), static_cast<int64_t>(B),
        beam_width, rp.preds.empty() ? nullptr : rp.preds.data(), static_cast<int32_t>(rp.preds.size()),
        rp.host.empty() ? nullptr : host_hook, &ctx, otok.data(), olp.data(), cnt.data(), st.data(), fp.data(),
        fs.data());
    if (!ctx.error.empty()) throw Error("predicate raised: " + ctx.error);
    check(s);
    BatchResult res;
    res.beams.resize(B);
    res.exhausted.resize(B);
    for (std::size_t b = 0; b < B; ++b) {
        if (st[b] != 0) {
            res.exhausted[b].exhausted = true;
            res.exhausted[b].step = fs[b];
            if (fp[b] >= 0 && static_cast<std::size_t>(fp[b]) < predicates.size())
                res.exhausted[b].predicate = predicates[static_cast<std::size_t>(fp[b])].name;
            continue;
        }
        for (int j = 0; j < cnt[b]; ++j) {
            ScoredSequence ss;
            ss.tokens.role = TokenSequence::Role::output;
            ss.tokens.ids.assign(otok.begin() + (b * k + j) * T, otok.begin() + (b * k + j + 1) * T);
            ss.log_prob = olp[b * k + j];
            res.beams[b].push_back(std::move(ss));
        }
    }
    return res;
}

std::vector<TokenSequence> greedy_decode_batch(const SequencePredictor& predictor,
                                               std::span<const TokenSequence> inputs) {
    const int T = predictor.num_positions();
    const std::size_t B = inputs.size();
    std::vector<int32_t> tok(B * 7), out(B * T);
    for (std::size_t b = 0; b < B; ++b) {
        if (inputs[b].length() != kNumInputFields)
            throw ParameterError("model input must have 7 tokens, got " + std::to_string(inputs[b].length()));
        for (int f = 0; f < 7; ++f) tok[b * 7 + f] = inputs[b].ids[static_cast<std::size_t>(f)];
    }
    check(ks_group_greedy_batch(predictor.group(), tok.data(), static_cast<int64_t>(B), out.data()));
    std::vector<TokenSequence> res(B);
    for (std::size_t b = 0; b < B; ++b) {
        res[b].role = TokenSequence::Role::output;
        res[b].ids.assign(out.begin() + b * T, out.begin() + (b + 1) * T);
    }
    return res;
}

TokenSequence greedy_decode(const SequencePredictor& predictor, const TokenSequence& input) {
    return greedy_decode_batch(predictor, std::span<const TokenSequence>(&input, 1))[0];
}

std::vector<ScoredSequence> beam_search(const SequencePredictor& predictor, const TokenSequence& input,
                                        int beam_width) {
    return beam_search_batch(predictor, std::span<const TokenSequence>(&input, 1), {}, beam_width, {}).beams[0];
}

std::vector<ScoredSequence> constrained_beam_search(const SequencePredictor& predictor, const TokenSequence& input,
                                                    int beam_width, std::span<const ConstraintPredicate> predicates,
                                                    const ProblemDescriptor& descriptor) {
    BatchResult r = beam_search_batch(predictor, std::span<const TokenSequence>(&input, 1),
                                      std::span<const ProblemDescriptor>(&descriptor, 1), beam_width, predicates);
    if (r.exhausted[0].exhausted) {
        const auto& e = r.exhausted[0];
        throw BeamExhaustedError("constrained beam search: every candidate at position " + std::to_string(e.step) +
                                     " was rejected (last rejecting predicate: " + e.predicate + ")",
                                 e.predicate, e.step);
    }
    return r.beams[0];
}

// ------------------------------------------------------------------ evaluation
EvalReport compute_metrics(const std::vector<TokenSequence>& predictions, const std::vector<TokenSequence>& actuals) {
    if (actuals.empty()) throw ParameterError("metrics: empty test set");
    if (predictions.size() != actuals.size())
        throw ParameterError("metrics: " + std::to_string(predictions.size()) + " predictions vs " +
                             std::to_string(actuals.size()) + " actuals");
    const std::size_t arity = actuals[0].ids.size();
    for (std::size_t i = 0; i < actuals.size(); ++i)
        if (predictions[i].ids.size() != arity || actuals[i].ids.size() != arity)
            throw ParameterError("metrics: sequences must have uniform arity");
    EvalReport r;
    r.sample_count = static_cast<int>(actuals.size());
    r.per_param_accuracy.assign(arity, 0.0);
    int perfect = 0;
    for (std::size_t i = 0; i < actuals.size(); ++i) {
        bool all = true;
        for (std::size_t p = 0; p < arity; ++p) {
            if (predictions[i].ids[p] == actuals[i].ids[p])
                r.per_param_accuracy[p] += 1.0;
            else
                all = false;
        }
        perfect += all ? 1 : 0;
    }
    const double S = static_cast<double>(actuals.size());
    double sum = 0.0;
    for (double& a : r.per_param_accuracy) {
        a = a / S * 100.0;
        sum += a;
    }
    r.average_accuracy = sum / static_cast<double>(arity);
    r.perfect_prediction = static_cast<double>(perfect) / S * 100.0;
    return r;
}

// topk_metrics (proj/src/eval.cpp:74-152): for each k a full batched search on
// the GPU; best-matching beam (most position matches, ties to the higher rank),
// perfect = any of the k beams equals the truth; exhausted searches score 0.
std::vector<EvalReport> topk_metrics(const ModelParams& params, const std::vector<Sample>& test,
                                     const std::vector<int>& k_values,
                                     std::span<const ConstraintPredicate> predicates, int threads) {
    const SequencePredictor predictor(params);
    return topk_metrics(predictor, test, k_values, predicates, threads);
}

std::vector<EvalReport> topk_metrics(const SequencePredictor& predictor, const std::vector<Sample>& test,
                                     const std::vector<int>& k_values,
                                     std::span<const ConstraintPredicate> predicates, int /*threads*/) {
    if (test.empty()) throw ParameterError("topk_metrics: empty test set");
    for (int k : k_values)
        if (k < 1) throw ParameterError("topk_metrics: k must be >= 1");
    const ModelParams& params = predictor.params();
    const KernelSpec spec = spec_of(params);
    const int arity = predictor.num_positions();
    const std::size_t B = test.size();
    std::vector<int32_t> tok(B * 7), truth(B * (size_t)arity);
    std::vector<int64_t> desc(B * 7);
    std::vector<ProblemDescriptor> descs;
    descs.reserve(B);
    for (std::size_t i = 0; i < B; ++i) {
        const TokenSequence in = encode_problem(test[i].descriptor, params.vocab);
        const TokenSequence tr = encode_params(test[i].params, spec, params.vocab);
        std::copy(in.ids.begin(), in.ids.end(), tok.begin() + (long)(i * 7));
        std::copy(tr.ids.begin(), tr.ids.end(), truth.begin() + (long)(i * (size_t)arity));
        for (int f = 0; f < 7; ++f) desc[i * 7 + (size_t)f] = descriptor_field(test[i].descriptor, f);
        descs.push_back(test[i].descriptor);
    }
    ResolvedPreds rp = resolve(params, predicates);
    // one device call for every k (a width-k search does not contain the width-j beams,
    // so each k is still its own search, as eval.cpp:74-152 runs them): each chunk is
    // encoded once and decoded at every width; the best-matching beam / any-of-k
    // scoring stays on the device
    const int nk = static_cast<int>(k_values.size());
    std::vector<int32_t> ks(k_values.begin(), k_values.end());
    std::vector<int64_t> hits((size_t)nk * (size_t)arity), perfect((size_t)nk);
    HookCtx ctx{&params, predicates, &rp.host, descs, {}};
    const ks_status s = ks_group_topk_metrics_multi(
        predictor.group(), tok.data(), desc.data(), truth.data(), static_cast<int64_t>(B), ks.data(), nk,
        rp.preds.empty() ? nullptr : rp.preds.data(), static_cast<int32_t>(rp.preds.size()),
        rp.host.empty() ? nullptr : host_hook, &ctx, hits.data(), perfect.data());
    if (!ctx.error.empty()) throw Error("predicate raised: " + ctx.error);
    check(s);
    std::vector<EvalReport> reports;
    for (int i = 0; i < nk; ++i) {
        EvalReport r;
        r.sample_count = static_cast<int>(B);
        r.per_param_accuracy.resize((size_t)arity);
        double sum = 0.0;
        for (int p = 0; p < arity; ++p) {
            r.per_param_accuracy[(size_t)p] =
                static_cast<double>(hits[(size_t)i * arity + p]) / static_cast<double>(B) * 100.0;
            sum += r.per_param_accuracy[(size_t)p];
        }
        r.average_accuracy = sum / arity;
        r.perfect_prediction = 100.0 * static_cast<double>(perfect[(size_t)i]) / static_cast<double>(B);
        r.beam_width = k_values[(size_t)i];
        r.constrained = !predicates.empty();
        reports.push_back(std::move(r));
    }
    return reports;
}

// ------------------------------------------------------------------ training
// Rng: mt19937_64 ([rand.eng.mers], parameters of std::mt19937_64) with the
// reference's SplitMix-style derive and 53-bit uniforms (rng.hpp:13-71).
Rng::Rng(std::uint64_t seed) {
    mt_[0] = seed;
    for (int i = 1; i < 312; ++i) mt_[i] = 6364136223846793005ULL * (mt_[i - 1] ^ (mt_[i - 1] >> 62)) + (std::uint64_t)i;
    idx_ = 312;
}

Rng Rng::derive(std::uint64_t seed, std::uint64_t stream) {
    auto mix = [](std::uint64_t z) {
        z += 0x9e3779b97f4a7c15ULL;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    };
    return Rng(mix(mix(seed) + 0x9e3779b97f4a7c15ULL * (stream + 1)));
}

std::uint64_t Rng::next_u64() {
    if (idx_ >= 312) {
        for (int i = 0; i < 312; ++i) {
            const std::uint64_t x = (mt_[i] & 0xFFFFFFFF80000000ULL) | (mt_[(i + 1) % 312] & 0x7FFFFFFFULL);
            std::uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            mt_[i] = mt_[(i + 156) % 312] ^ xa;
        }
        idx_ = 0;
    }
    std::uint64_t y = mt_[idx_++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

double Rng::uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }

std::uint64_t Rng::uniform_int(std::uint64_t n) {
    const std::uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    std::uint64_t v;
    do {
        v = next_u64();
    } while (v >= limit);
    return v % n;
}

// build_vocab (encoding.cpp:52-86): input values seen per field, ascending;
// outputs are the spec's legal sets.
Vocabulary build_vocab(const KernelSpec& spec, const std::vector<Sample>& dataset) {
    if (dataset.empty()) throw ParameterError("build_vocab: dataset is empty");
    std::array<std::vector<std::int64_t>, kNumInputFields> seen;
    for (const Sample& smp : dataset) {
        for (int f = 0; f < kNumInputFields; ++f) seen[(size_t)f].push_back(descriptor_field(smp.descriptor, f));
        for (const auto& p : spec.params) {
            auto it = smp.params.find(p.name);
            if (it == smp.params.end()) throw ValidationError("sample missing parameter " + p.name, p.name);
            if (std::find(p.values.begin(), p.values.end(), it->second) == p.values.end())
                throw ValidationError("value " + std::to_string(it->second) + " of parameter " + p.name +
                                          " is outside the legal set for kernel " + spec.name,
                                      p.name);
        }
    }
    std::vector<FieldVocab> in, out;
    for (int f = 0; f < kNumInputFields; ++f) {
        auto& v = seen[(size_t)f];
        std::sort(v.begin(), v.end());
        v.erase(std::unique(v.begin(), v.end()), v.end());
        in.push_back({kInputFieldNames[(size_t)f], v});
    }
    for (const auto& p : spec.params) out.push_back({p.name, p.values});
    return Vocabulary(std::move(in), std::move(out));
}

namespace {

int feedback_width(const Vocabulary& v) {
    int w = 1;  // GO slot
    for (const auto& f : v.output_params()) w += f.size();
    return w;
}
int input_width(const Vocabulary& v) {
    int w = 0;
    for (const auto& f : v.input_fields()) w += f.size();
    return w;
}

// nn::lstm_init (nn.cpp:309-318): w_* (in + H) x H ~ U(-1/sqrt(H), 1/sqrt(H)) drawn
// in the order input, forget, output, cand; forget bias 1.
void put_lstm_init(ModelParams& mp, const std::string& prefix, int in, int H, Rng& rng) {
    const double lim = 1.0 / std::sqrt(static_cast<double>(H));
    static const char* gates[4] = {"input", "forget", "output", "cand"};
    for (const char* g : gates) {
        HostTensor w;
        w.shape = {in + H, H};
        w.values.resize((size_t)(in + H) * H);
        for (auto& x : w.values) x = static_cast<float>(rng.uniform(-lim, lim));
        mp.tensors[prefix + ".w_" + g] = std::move(w);
    }
    for (const char* g : gates) {
        HostTensor b;
        b.shape = {H};
        b.values.assign((size_t)H, std::string(g) == "forget" ? 1.0f : 0.0f);
        mp.tensors[prefix + ".b_" + g] = std::move(b);
    }
}

// nn::xavier_uniform / dense_init (nn.cpp:299-329)
void put_dense_init(ModelParams& mp, const std::string& prefix, int in, int out, Rng& rng) {
    const double lim = std::sqrt(6.0 / (in + out));
    HostTensor w;
    w.shape = {in, out};
    w.values.resize((size_t)in * out);
    for (auto& x : w.values) x = static_cast<float>(rng.uniform(-lim, lim));
    mp.tensors[prefix + ".weights"] = std::move(w);
    HostTensor b;
    b.shape = {out};
    b.values.assign((size_t)out, 0.0f);
    mp.tensors[prefix + ".bias"] = std::move(b);
}

}  // namespace

// init_model (models.cpp:178-259): same tensor names, shapes and draw order from
// Rng::derive(seed, 0x171); values rounded to fp32 as a checkpoint stores them.
ModelParams init_model(const ModelConfig& config, const KernelSpec& spec, const Vocabulary& vocab,
                       Precision precision, std::uint64_t seed) {
    spec.check();
    if (vocab.num_output_positions() != spec.num_params())
        throw ParameterError("vocabulary has " + std::to_string(vocab.num_output_positions()) +
                             " output positions, kernel " + spec.name + " has " + std::to_string(spec.num_params()));
    ModelParams mp;
    mp.config = config;
    mp.kernel = spec.name;
    mp.precision = precision;
    mp.vocab = vocab;
    Rng rng = Rng::derive(seed, 0x171);
    const int d_in = input_width(vocab), d_fb = feedback_width(vocab), T = vocab.num_output_positions();
    int head_in = 0;
    switch (config.variant) {
        case ModelVariant::enc_dec:
            put_lstm_init(mp, "encoder", d_in, config.encoder_state_size, rng);
            put_lstm_init(mp, "decoder", d_fb, config.encoder_state_size, rng);
            head_in = config.encoder_state_size;
            break;
        case ModelVariant::attn:
        case ModelVariant::attn2: {
            put_lstm_init(mp, "pre.fwd", d_in, config.pre_attention_size, rng);
            put_lstm_init(mp, "pre.bwd", d_in, config.pre_attention_size, rng);
            const int act = 2 * config.pre_attention_size;
            put_lstm_init(mp, "post", config.variant == ModelVariant::attn ? act + d_fb : act, config.post_attention_size,
                          rng);
            put_dense_init(mp, "attn.hidden", config.post_attention_size + act, config.attention_dense_nodes, rng);
            put_dense_init(mp, "attn.out", config.attention_dense_nodes, 1, rng);
            head_in = config.post_attention_size;
            break;
        }
        case ModelVariant::hybrid:
        case ModelVariant::hybrid2: {
            if (config.conv_layers.empty()) throw ParameterError("hybrid variants need at least one conv layer");
            int ch = d_in, len = kNumInputFields;
            for (std::size_t i = 0; i < config.conv_layers.size(); ++i) {
                const ConvLayerSpec& l = config.conv_layers[i];
                if (len < l.kernel_size) throw ShapeError("conv stack input length shorter than kernel size");
                const int fan_in = ch * l.kernel_size, fan_out = l.filters * l.kernel_size;
                const double lim = std::sqrt(6.0 / (fan_in + fan_out));
                HostTensor f;
                f.shape = {l.filters, ch, l.kernel_size};
                f.values.resize((size_t)l.filters * ch * l.kernel_size);
                for (auto& x : f.values) x = static_cast<float>(rng.uniform(-lim, lim));
                mp.tensors["conv." + std::to_string(i) + ".filters"] = std::move(f);
                HostTensor b;
                b.shape = {l.filters};
                b.values.assign((size_t)l.filters, 0.0f);
                mp.tensors["conv." + std::to_string(i) + ".bias"] = std::move(b);
                len = (len - l.kernel_size) / l.stride + 1;
                ch = l.filters;
            }
            const int flat = ch * len, cell = config.decoder_cell_size;
            put_lstm_init(mp, "bilstm1.fwd", flat, cell, rng);
            put_lstm_init(mp, "bilstm1.bwd", flat, cell, rng);
            const int b2 = config.variant == ModelVariant::hybrid ? 2 * cell : flat;
            put_lstm_init(mp, "bilstm2.fwd", b2, cell, rng);
            put_lstm_init(mp, "bilstm2.bwd", b2, cell, rng);
            head_in = 2 * cell;
            break;
        }
    }
    for (int i = 0; i < T; ++i) put_dense_init(mp, "head." + std::to_string(i), head_in, vocab.output_param(i).size(), rng);
    return mp;
}

// save_checkpoint (data.cpp:464-509): kernelseer-checkpoint/1.
void save_checkpoint(const ModelParams& params, const std::string& path) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw CheckpointError(CheckpointError::Kind::io, "cannot write " + path);
    const ModelConfig& c = params.config;
    out << "format: kernelseer-checkpoint/1\n";
    out << "variant: " << variant_label(c.variant) << "\n";
    out << "kernel: " << params.kernel << "\n";
    out << "precision: " << precision_label(params.precision) << "\n";
    out << "encoder_state_size: " << c.encoder_state_size << "\n";
    out << "pre_attention_size: " << c.pre_attention_size << "\n";
    out << "post_attention_size: " << c.post_attention_size << "\n";
    out << "attention_dense_nodes: " << c.attention_dense_nodes << "\n";
    out << "decoder_cell_size: " << c.decoder_cell_size << "\n";
    out << "dropout: " << c.dropout << "\n";
    out << "recurrent_dropout: " << c.recurrent_dropout << "\n";
    out << "conv_layers: ";
    for (std::size_t i = 0; i < c.conv_layers.size(); ++i)
        out << (i ? ";" : "") << c.conv_layers[i].filters << "," << c.conv_layers[i].kernel_size << ","
            << c.conv_layers[i].stride;
    out << "\n";
    for (int f = 0; f < kNumInputFields; ++f)
        out << "input_vocab." << params.vocab.input_field(f).name << ": " << join(params.vocab.input_field(f).values)
            << "\n";
    out << "output_params: " << params.vocab.num_output_positions() << "\n";
    for (int i = 0; i < params.vocab.num_output_positions(); ++i)
        out << "param." << i << ": " << params.vocab.output_param(i).name << " = "
            << join(params.vocab.output_param(i).values) << "\n";
    for (const auto& [name, t] : params.tensors) {
        out << "tensor: " << name << " ";
        for (std::size_t i = 0; i < t.shape.size(); ++i) out << (i ? "x" : "") << t.shape[i];
        out << "\n";
    }
    out << "\n";
    for (const auto& [name, t] : params.tensors) {
        for (float v : t.values) {
            std::uint32_t u;
            std::memcpy(&u, &v, 4);
            const unsigned char b[4] = {(unsigned char)(u & 0xFF), (unsigned char)((u >> 8) & 0xFF),
                                        (unsigned char)((u >> 16) & 0xFF), (unsigned char)(u >> 24)};
            out.write(reinterpret_cast<const char*>(b), 4);
        }
    }
    if (!out) throw CheckpointError(CheckpointError::Kind::io, "write failed: " + path);
}

namespace {

// The flattened ModelParams a ks_model_desc points into.
struct DescHolder {
    std::vector<int32_t> in_sizes, vsizes, conv;
    std::vector<int64_t> in_vals, out_vals;
    std::vector<const char*> names;
    std::vector<int32_t> numel;
    std::vector<const float*> data;
    ks_model_desc d{};
    explicit DescHolder(const ModelParams& params) {
        for (const auto& f : params.vocab.input_fields()) {
            in_sizes.push_back(f.size());
            in_vals.insert(in_vals.end(), f.values.begin(), f.values.end());
        }
        for (const auto& f : params.vocab.output_params()) {
            vsizes.push_back(f.size());
            out_vals.insert(out_vals.end(), f.values.begin(), f.values.end());
        }
        for (const auto& [n, t] : params.tensors) {
            names.push_back(n.c_str());
            numel.push_back(static_cast<int32_t>(t.values.size()));
            data.push_back(t.values.data());
        }
        for (const auto& l : params.config.conv_layers) {
            conv.push_back(l.filters);
            conv.push_back(l.kernel_size);
            conv.push_back(l.stride);
        }
        d.variant = static_cast<int32_t>(params.config.variant);
        d.decoder_cell_size = params.config.decoder_cell_size;
        d.num_conv_layers = static_cast<int32_t>(params.config.conv_layers.size());
        d.conv_layers = conv.data();
        d.encoder_state_size = params.config.encoder_state_size;
        d.pre_attention_size = params.config.pre_attention_size;
        d.post_attention_size = params.config.post_attention_size;
        d.attention_dense_nodes = params.config.attention_dense_nodes;
        d.num_positions = params.num_output_positions();
        d.input_sizes = in_sizes.data();
        d.input_values = in_vals.data();
        d.vocab_sizes = vsizes.data();
        d.output_values = out_vals.data();
        d.num_tensors = static_cast<int32_t>(names.size());
        d.tensor_names = names.data();
        d.tensor_numel = numel.data();
        d.tensor_data = data.data();
    }
};

}  // namespace

// train_model (models.cpp:862-969): init_model, per epoch a Fisher-Yates shuffle
// from Rng::derive(seed, 0x3ff000 + epoch), batches of batch_size in that order
// (each sample's dropout stream Rng::derive(seed, epoch << 32 | index) drawn on the
// device), gradient sum / batch, clip, Adam; then the test set teacher-forced
// (dropout off).  One GPU; data-parallel training is paper_2404_10162_b200.train.
TrainResult train_model(const ModelConfig& config, const KernelSpec& spec, const Vocabulary& vocab,
                        Precision precision, const std::vector<Sample>& train_set,
                        const std::vector<Sample>& test_set, const TrainOptions& options,
                        const std::function<void(const EpochStats&)>& on_epoch, int device) {
    if (train_set.empty()) throw ParameterError("train_model: empty training set");
    if (options.epochs < 1 || options.batch_size < 1)
        throw ParameterError("train_model: epochs and batch size must be >= 1");
    if (config.dropout < 0.0 || config.dropout >= 1.0 || config.recurrent_dropout < 0.0 ||
        config.recurrent_dropout >= 1.0)
        throw ParameterError("dropout rates must be in [0,1)");
    const int T = vocab.num_output_positions();
    auto encode_all = [&](const std::vector<Sample>& set, std::vector<int32_t>& tok, std::vector<int32_t>& tgt) {
        for (const Sample& smp : set) {
            const TokenSequence in = encode_problem(smp.descriptor, vocab);
            const TokenSequence out = encode_params(smp.params, spec, vocab);
            tok.insert(tok.end(), in.ids.begin(), in.ids.end());
            tgt.insert(tgt.end(), out.ids.begin(), out.ids.end());
        }
    };
    std::vector<int32_t> tr_tok, tr_tgt, te_tok, te_tgt;
    encode_all(train_set, tr_tok, tr_tgt);
    encode_all(test_set, te_tok, te_tgt);

    TrainResult result;
    result.params = init_model(config, spec, vocab, precision, options.seed);
    ks_trainer* tr = nullptr;
    {
        DescHolder h(result.params);
        check(ks_trainer_create(&h.d, config.dropout, config.recurrent_dropout, device, &tr));
    }
    std::unique_ptr<ks_trainer, void (*)(ks_trainer*)> guard(tr, ks_trainer_destroy);
    const int n = static_cast<int>(train_set.size());
    std::vector<int32_t> btok, btgt;
    std::vector<int64_t> bidx;
    for (int epoch = 1; epoch <= options.epochs; ++epoch) {
        std::vector<int> order((size_t)n);
        for (int i = 0; i < n; ++i) order[(size_t)i] = i;
        Rng shuffle = Rng::derive(options.seed, 0x3ff000ULL + static_cast<std::uint64_t>(epoch));
        for (std::size_t i = order.size(); i > 1; --i) std::swap(order[i - 1], order[shuffle.uniform_int(i)]);
        double epoch_loss = 0.0;
        long long matches = 0;
        for (int start = 0; start < n; start += options.batch_size) {
            const int B = std::min(n, start + options.batch_size) - start;
            btok.resize((size_t)B * kNumInputFields);
            btgt.resize((size_t)B * T);
            bidx.resize((size_t)B);
            for (int b = 0; b < B; ++b) {
                const int idx = order[(size_t)(start + b)];
                std::memcpy(&btok[(size_t)b * kNumInputFields], &tr_tok[(size_t)idx * kNumInputFields],
                            sizeof(int32_t) * kNumInputFields);
                std::memcpy(&btgt[(size_t)b * T], &tr_tgt[(size_t)idx * T], sizeof(int32_t) * (size_t)T);
                bidx[(size_t)b] = idx;
            }
            double loss = 0.0;
            int64_t m = 0;
            check(ks_trainer_step(tr, btok.data(), btgt.data(), bidx.data(), B, epoch, options.seed,
                                  options.learning_rate, options.clip_norm, &loss, &m));
            epoch_loss += loss;
            matches += m;
        }
        EpochStats st;
        st.epoch = epoch;
        st.train_loss = epoch_loss / n;
        st.train_accuracy = 100.0 * static_cast<double>(matches) / (static_cast<double>(n) * T);
        if (!test_set.empty()) {
            double loss = 0.0;
            int64_t m = 0;
            check(ks_trainer_evaluate(tr, te_tok.data(), te_tgt.data(), (int64_t)test_set.size(), &loss, &m));
            st.test_loss = loss / static_cast<double>(test_set.size());
            st.test_accuracy = 100.0 * static_cast<double>(m) / (static_cast<double>(test_set.size()) * T);
        }
        result.log.push_back(st);
        if (on_epoch) on_epoch(st);
    }
    // trained parameters back into the reference tensors (checkpoint order)
    std::vector<float> flat((size_t)ks_trainer_num_ref_params(tr));
    check(ks_trainer_export(tr, flat.data()));
    std::size_t o = 0;
    for (auto& [name, t] : result.params.tensors) {
        std::copy(flat.begin() + (long)o, flat.begin() + (long)(o + t.values.size()), t.values.begin());
        o += t.values.size();
    }
    return result;
}

}  // namespace kernelseer
