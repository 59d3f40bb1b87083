// Test infrastructure (oracle/): an extern "C" driver over the UNMODIFIED
// reference core (compiled from /root/reference/proj/src by oracle/Makefile).
// It is the "reference" CPU arm of bench.py and a checker for tests; it is
// never linked into, or called by, the product.
//
// Batching mirrors the reference's own batched caller: topk_metrics stripes
// samples over std::threads (proj/src/eval.cpp:105-137 via
// proj/include/kernelseer/parallel.hpp:14-27) and calls beam_search /
// constrained_beam_search per sample (proj/src/decoding.cpp:126-135).
#include <atomic>
#include <optional>
#include <stdexcept>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "kernelseer/data.hpp"
#include "kernelseer/decoding.hpp"
#include "kernelseer/eval.hpp"
#include "kernelseer/models.hpp"
#include "kernelseer/nn.hpp"
#include "kernelseer/parallel.hpp"
#include "kernelseer/rng.hpp"

using namespace kernelseer;
using kernelseer::nn::Tensor;

namespace {
thread_local std::string g_err;

// Predicate program text, one predicate per line:
//   membership                      -> membership_predicate(spec_of(model))
//   budget <name> <budget> p=w,...  -> resource_budget_predicate(weights, budget, name)
std::vector<ConstraintPredicate> parse_preds(const ModelParams& mp, const char* text) {
    std::vector<ConstraintPredicate> out;
    if (!text) return out;
    std::stringstream ss(text);
    std::string line;
    while (std::getline(ss, line)) {
        if (line.empty()) continue;
        std::stringstream ls(line);
        std::string kind;
        ls >> kind;
        if (kind == "membership") {
            out.push_back(membership_predicate(spec_of(mp)));
        } else if (kind == "budget") {
            std::string name, ws;
            double budget = 0;
            ls >> name >> budget >> ws;
            std::map<std::string, double> weights;
            std::stringstream wss(ws);
            std::string kv;
            while (std::getline(wss, kv, ',')) {
                auto eq = kv.find('=');
                if (eq == std::string::npos) continue;
                weights[kv.substr(0, eq)] = std::stod(kv.substr(eq + 1));
            }
            out.push_back(resource_budget_predicate(weights, budget, name));
        } else {
            throw ParameterError("ref_shim: unknown predicate kind " + kind);
        }
    }
    return out;
}

ProblemDescriptor desc_of(const int64_t* d) {
    ProblemDescriptor p;
    p.n = d[0]; p.c = d[1]; p.h_i = d[2]; p.w_i = d[3]; p.k = d[4]; p.y = d[5]; p.x = d[6];
    return p;
}
}  // namespace

extern "C" {

const char* ksref_last_error() { return g_err.c_str(); }

void* ksref_load(const char* path) {
    try {
        return new ModelParams(load_checkpoint(path));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ksref_free(void* h) { delete static_cast<ModelParams*>(h); }

int ksref_num_positions(void* h) { return static_cast<ModelParams*>(h)->num_output_positions(); }

int ksref_vocab_size(void* h, int pos) {
    return static_cast<ModelParams*>(h)->vocab.output_param(pos).size();
}

// Encodes descriptors (B x 7 int64) to token ids (B x 7 int32); -1 row on error.
int ksref_encode(void* h, const int64_t* desc, int64_t B, int32_t* tok) {
    const ModelParams& mp = *static_cast<ModelParams*>(h);
    int bad = 0;
    for (int64_t b = 0; b < B; ++b) {
        try {
            TokenSequence t = encode_problem(desc_of(desc + 7 * b), mp.vocab, false);
            for (int f = 0; f < 7; ++f) tok[7 * b + f] = t.ids[f];
        } catch (const std::exception&) {
            for (int f = 0; f < 7; ++f) tok[7 * b + f] = -1;
            ++bad;
        }
    }
    return bad;
}

// encode_problem with the allow_nearest snap (encoding.cpp:87-113) for each of B
// descriptors: tok B x 7 (-1 row on error), err_field B x 16 chars ("" when ok).
int ksref_encode_ex(void* h, const int64_t* desc, int64_t B, int allow_nearest, int32_t* tok, char* err_field) {
    const ModelParams& mp = *static_cast<ModelParams*>(h);
    int bad = 0;
    for (int64_t b = 0; b < B; ++b) {
        err_field[16 * b] = 0;
        try {
            TokenSequence t = encode_problem(desc_of(desc + 7 * b), mp.vocab, allow_nearest != 0);
            for (int f = 0; f < 7; ++f) tok[7 * b + f] = t.ids[f];
        } catch (const ValidationError& e) {
            for (int f = 0; f < 7; ++f) tok[7 * b + f] = -1;
            std::snprintf(err_field + 16 * b, 16, "%s", e.field().c_str());
            ++bad;
        }
    }
    return bad;
}

// Batched (constrained) beam search.  out_tok: B x k x T, out_lp: B x k,
// out_count: B, out_status: B (0 ok, 1 exhausted, 2 other error),
// out_fail_step: B, out_fail_name: B x 64 chars.
int ksref_beam_batch(void* h, const int32_t* tok, const int64_t* desc, int64_t B, int k,
                     const char* preds_text, int threads, int32_t* out_tok, double* out_lp,
                     int32_t* out_count, int32_t* out_status, int32_t* out_fail_step,
                     char* out_fail_name) {
    try {
        const ModelParams& mp = *static_cast<ModelParams*>(h);
        const std::vector<ConstraintPredicate> preds = parse_preds(mp, preds_text);
        const SequencePredictor predictor(mp);
        const int T = predictor.num_positions();
        parallel_stripes(static_cast<int>(B), threads, [&](int w, int stride) {
            for (int64_t b = w; b < B; b += stride) {
                TokenSequence in;
                in.ids.assign(tok + 7 * b, tok + 7 * b + 7);
                out_count[b] = 0;
                out_status[b] = 0;
                out_fail_step[b] = -1;
                if (out_fail_name) out_fail_name[64 * b] = 0;
                try {
                    std::vector<ScoredSequence> beams =
                        preds.empty() ? beam_search(predictor, in, k)
                                      : constrained_beam_search(predictor, in, k, preds,
                                                                desc_of(desc + 7 * b));
                    out_count[b] = static_cast<int32_t>(beams.size());
                    for (size_t j = 0; j < beams.size(); ++j) {
                        out_lp[b * k + j] = beams[j].log_prob;
                        for (int t = 0; t < T; ++t)
                            out_tok[(b * k + j) * T + t] = beams[j].tokens.ids[t];
                    }
                } catch (const BeamExhaustedError& e) {
                    out_status[b] = 1;
                    out_fail_step[b] = e.step();
                    if (out_fail_name) {
                        std::strncpy(out_fail_name + 64 * b, e.predicate().c_str(), 63);
                        out_fail_name[64 * b + 63] = 0;
                    }
                } catch (const std::exception&) {
                    out_status[b] = 2;
                }
            }
        });
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

int ksref_greedy_batch(void* h, const int32_t* tok, int64_t B, int threads, int32_t* out_tok) {
    try {
        const ModelParams& mp = *static_cast<ModelParams*>(h);
        const SequencePredictor predictor(mp);
        const int T = predictor.num_positions();
        parallel_stripes(static_cast<int>(B), threads, [&](int w, int stride) {
            for (int64_t b = w; b < B; b += stride) {
                TokenSequence in;
                in.ids.assign(tok + 7 * b, tok + 7 * b + 7);
                TokenSequence out = greedy_decode(predictor, in);
                for (int t = 0; t < T; ++t) out_tok[b * T + t] = out.ids[t];
            }
        });
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Teacher-forced per-position distributions (model_forward, proj/src/models.cpp:495-514):
// out: sum_p V_p doubles.
int ksref_forward(void* h, const int32_t* tok, const int32_t* teacher, double* out) {
    try {
        const ModelParams& mp = *static_cast<ModelParams*>(h);
        TokenSequence in;
        in.ids.assign(tok, tok + 7);
        const int T = mp.num_output_positions();
        std::vector<int> t(teacher, teacher + T);
        const auto dists = model_forward(mp, in, teacher ? &t : nullptr);
        size_t o = 0;
        for (const auto& d : dists)
            for (int i = 0; i < d.size(); ++i) out[o++] = d[i];
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// init_model over a synthetic vocabulary, then save_checkpoint (fp32 payload).
int ksref_init_save(const char* variant, int e_size, int n_a, int n_s, int n_d, int cell,
                    const char* kernel, int synth_count, uint64_t synth_seed,
                    const char* difficulty, uint64_t init_seed, const char* path) {
    try {
        const KernelSpec& spec = builtin_spec(kernel);
        const Dataset ds = generate_synthetic(spec, synth_count, synth_seed,
                                              difficulty_from_label(difficulty));
        const Vocabulary vocab = build_vocab(spec, ds.samples);
        ModelConfig c;
        c.variant = variant_from_label(variant);
        c.encoder_state_size = e_size;
        c.pre_attention_size = n_a;
        c.post_attention_size = n_s;
        c.attention_dense_nodes = n_d;
        c.decoder_cell_size = cell;
        c.dropout = 0.0;
        c.recurrent_dropout = 0.0;
        const ModelParams mp = init_model(c, spec, vocab, Precision::full, init_seed);
        save_checkpoint(mp, path);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// init_model over a custom spec line ("K|p0=0-2|p1=0,1") with every input
// field's vocabulary {1, 2}: the tiny_model fixture of proj/tests/test_util.hpp:50-88.
int ksref_init_save_spec(const char* variant, int cell, const char* spec_line, uint64_t seed,
                         const char* path) {
    try {
        const KernelSpec spec = parse_kernel_spec_line(spec_line);
        std::vector<FieldVocab> inputs;
        for (int f = 0; f < kNumInputFields; ++f)
            inputs.push_back(FieldVocab{kInputFieldNames[static_cast<std::size_t>(f)], {1, 2}});
        std::vector<FieldVocab> outputs;
        for (const auto& p : spec.params) outputs.push_back(FieldVocab{p.name, p.values});
        const Vocabulary vocab(std::move(inputs), std::move(outputs));
        ModelConfig c;
        c.variant = variant_from_label(variant);
        c.encoder_state_size = cell;
        c.pre_attention_size = cell;
        c.post_attention_size = cell;
        c.attention_dense_nodes = 2;
        c.decoder_cell_size = cell;
        c.conv_layers = {{4, 3, 1}, {3, 3, 1}};
        c.dropout = 0.0;
        c.recurrent_dropout = 0.0;
        const ModelParams mp = init_model(c, spec, vocab, Precision::full, seed);
        save_checkpoint(mp, path);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Synthetic descriptors exactly as generate_synthetic draws them (unique grid
// points, proj/src/data.cpp:348-395): out B x 7 int64.
int ksref_synthetic(const char* kernel, int count, uint64_t seed, const char* difficulty,
                    int64_t* out_desc, int32_t* out_params /* count x T token ids or null */) {
    try {
        const KernelSpec& spec = builtin_spec(kernel);
        const Dataset ds = generate_synthetic(spec, count, seed, difficulty_from_label(difficulty));
        for (int i = 0; i < count; ++i) {
            const ProblemDescriptor& d = ds.samples[i].descriptor;
            const int64_t v[7] = {d.n, d.c, d.h_i, d.w_i, d.k, d.y, d.x};
            for (int f = 0; f < 7; ++f) out_desc[7 * i + f] = v[f];
            if (out_params) {
                for (int p = 0; p < spec.num_params(); ++p) {
                    const auto& vals = spec.params[p].values;
                    const int64_t val = ds.samples[i].params.at(spec.params[p].name);
                    int id = -1;
                    for (size_t j = 0; j < vals.size(); ++j)
                        if (vals[j] == val) id = static_cast<int>(j);
                    out_params[i * spec.num_params() + p] = id;
                }
            }
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Benchmark / parity workloads drawn with the reference's own Rng (rng.hpp:19-43):
// config start+i draws each input field uniformly with replacement from the model's
// input vocabulary, fields in order n,c,h,w,k,y,x, from Rng::derive(seed, start+i).
// The checker for ks_synthetic_descriptors.
int ksref_descriptors(void* h, uint64_t seed, int64_t start, int64_t count, int64_t* out) {
    try {
        const ModelParams& mp = *static_cast<ModelParams*>(h);
        for (int64_t i = 0; i < count; ++i) {
            Rng r = Rng::derive(seed, static_cast<std::uint64_t>(start + i));
            for (int f = 0; f < kNumInputFields; ++f) {
                const auto& vals = mp.vocab.input_field(f).values;
                out[7 * i + f] = vals[static_cast<std::size_t>(r.uniform_int(vals.size()))];
            }
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// ---------------------------------------------------------------------------
// Teacher-forced training (BASELINE config 4), reference side.
// ---------------------------------------------------------------------------

// Flat gradient / parameter layout: the tensors in ModelParams::tensors order
// (std::map = alphabetical = checkpoint payload order, proj/src/data.cpp:497-509).
int64_t ksref_num_params(void* h) {
    int64_t n = 0;
    for (const auto& [name, t] : static_cast<ModelParams*>(h)->tensors) n += t.size();
    return n;
}

int ksref_get_params(void* h, double* out) {
    int64_t o = 0;
    for (const auto& [name, t] : static_cast<ModelParams*>(h)->tensors)
        for (int i = 0; i < t.size(); ++i) out[o++] = t[i];
    return 0;
}

// Sum over samples of model_loss_gradients (proj/src/models.cpp:788-797).
// dropout_epoch < 0: no dropout (rng = nullptr).  Otherwise each sample b gets
// the stream train_model gives it: Rng::derive(seed, epoch << 32 | idx[b])
// (proj/src/models.cpp:915-918).  grads: flat, ksref_num_params doubles.
int ksref_loss_grads(void* h, const int32_t* tok, const int32_t* tgt, int64_t B, int threads,
                     int64_t dropout_epoch, uint64_t seed, const int64_t* idx, double* loss_sum,
                     double* grads) {
    try {
        const ModelParams& mp = *static_cast<ModelParams*>(h);
        const int T = mp.num_output_positions();
        threads = std::max(1, threads);
        std::vector<std::map<std::string, Tensor>> part(static_cast<size_t>(threads));
        std::vector<double> ploss(static_cast<size_t>(threads), 0.0);
        std::vector<std::string> errs(static_cast<size_t>(threads));
        parallel_stripes(static_cast<int>(B), threads, [&](int w, int stride) {
            try {
                for (int64_t b = w; b < B; b += stride) {
                    TokenSequence in, out;
                    in.ids.assign(tok + 7 * b, tok + 7 * b + 7);
                    out.ids.assign(tgt + T * b, tgt + T * b + T);
                    std::optional<Rng> rng;
                    if (dropout_epoch >= 0)
                        rng.emplace(Rng::derive(seed, (static_cast<uint64_t>(dropout_epoch) << 32) |
                                                          static_cast<uint64_t>(idx ? idx[b] : b)));
                    auto [loss, g] = model_loss_gradients(mp, in, out, rng ? &*rng : nullptr);
                    ploss[w] += loss;
                    auto& acc = part[static_cast<size_t>(w)];
                    for (auto& [name, t] : g) {
                        auto it = acc.find(name);
                        if (it == acc.end()) acc.emplace(name, t);
                        else for (int i = 0; i < t.size(); ++i) it->second[i] += t[i];
                    }
                }
            } catch (const std::exception& e) {
                errs[static_cast<size_t>(w)] = e.what();
            }
        });
        for (const auto& e : errs)
            if (!e.empty()) throw std::runtime_error(e);
        double ls = 0.0;
        for (double l : ploss) ls += l;
        if (loss_sum) *loss_sum = ls;
        int64_t o = 0;
        for (const auto& [name, t] : mp.tensors) {
            for (int i = 0; i < t.size(); ++i) {
                double v = 0.0;
                for (const auto& pm : part) {
                    auto it = pm.find(name);
                    if (it != pm.end()) v += it->second[i];
                }
                grads[o++] = v;
            }
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// One optimiser step of train_model's batch loop (proj/src/models.cpp:905-947):
// summed per-sample grads (dropout streams as train_model), / batch,
// clip_global_norm, adam_step.  The Adam state lives in the handle's trainer.
struct RefTrainer {
    nn::AdamState adam;
};

void* ksref_trainer_new(double lr) {
    auto* t = new RefTrainer();
    t->adam.config.learning_rate = lr;
    return t;
}
void ksref_trainer_free(void* t) { delete static_cast<RefTrainer*>(t); }

int ksref_train_step(void* h, void* trainer, const int32_t* tok, const int32_t* tgt, int64_t B,
                     int threads, int64_t epoch, uint64_t seed, const int64_t* idx, double clip,
                     double* loss_sum) {
    try {
        ModelParams& mp = *static_cast<ModelParams*>(h);
        const int64_t n = ksref_num_params(h);
        std::vector<double> g(static_cast<size_t>(n));
        const bool drop = mp.config.dropout != 0.0 || mp.config.recurrent_dropout != 0.0;
        if (ksref_loss_grads(h, tok, tgt, B, threads, drop ? epoch : -1, seed, idx, loss_sum, g.data()))
            return -1;
        std::map<std::string, Tensor> grads;
        int64_t o = 0;
        for (const auto& [name, t] : mp.tensors) {
            Tensor gt(t.shape());
            for (int i = 0; i < gt.size(); ++i) gt[i] = g[static_cast<size_t>(o++)] / static_cast<double>(B);
            grads.emplace(name, std::move(gt));
        }
        nn::clip_global_norm(grads, clip);
        nn::adam_step(mp.tensors, grads, static_cast<RefTrainer*>(trainer)->adam);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

int ksref_save(void* h, const char* path) {
    try {
        save_checkpoint(*static_cast<ModelParams*>(h), path);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Rng streams as the reference draws them (proj/include/kernelseer/rng.hpp).
void ksref_uniforms(uint64_t seed, uint64_t stream, int64_t n, double* out) {
    Rng r = Rng::derive(seed, stream);
    for (int64_t i = 0; i < n; ++i) out[i] = r.uniform();
}

void ksref_shuffle(uint64_t seed, uint64_t epoch, int64_t n, int64_t* order) {
    for (int64_t i = 0; i < n; ++i) order[i] = i;
    Rng r = Rng::derive(seed, 0x3ff000ULL + epoch);
    for (int64_t i = n; i > 1; --i) std::swap(order[i - 1], order[r.uniform_int(static_cast<uint64_t>(i))]);
}

}  // extern "C"
