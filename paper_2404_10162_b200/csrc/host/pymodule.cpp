// pymodule.cpp -- the Python face of the engine: the same function names,
// keyword arguments and return shapes as the reference's pybind module
// (proj/bindings/module.cpp:106-355) for the decode path, implemented on the
// C++ host layer (kernelseer_b200.hpp) and therefore on the GPU.
//
// Differences that are deliberate:
//  * the GIL is released around every device call (the reference holds it,
//    which deadlocks topk_metrics(threads>1) with Python predicates);
//  * ModelParams caches its device engine (weights packed once per process);
//  * predict_batch / greedy_predict_batch take many descriptors in one call.
#include <pybind11/functional.h>
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <mutex>
#include <optional>
#include <tuple>

#include "kernelseer_b200.hpp"
#include "ks_b200.h"

namespace py = pybind11;
using namespace kernelseer;

namespace {

struct PyModel {
    std::shared_ptr<ModelParams> params;
    std::shared_ptr<SequencePredictor> predictor;
    int device = SequencePredictor::kAllDevices;  // every visible GPU (set_engine narrows it)
    std::vector<int> devices;                     // explicit device list (set_engine([...]))
    GemmPrecision precision = GemmPrecision::f16x3;
    std::mutex mu;
    const SequencePredictor& pred() {
        std::lock_guard<std::mutex> g(mu);
        if (!predictor)
            predictor = devices.empty() ? std::make_shared<SequencePredictor>(*params, device, precision)
                                        : std::make_shared<SequencePredictor>(*params, devices, precision);
        return *predictor;
    }
};

ProblemDescriptor descriptor_from_dict(const py::dict& d) {
    ProblemDescriptor out;
    for (auto item : d) {
        const std::string key = py::cast<std::string>(item.first);
        if (key == "precision") {
            out.precision = precision_from_label(py::cast<std::string>(item.second));
            continue;
        }
        bool known = false;
        for (int f = 0; f < kNumInputFields; ++f)
            if (key == kInputFieldNames[static_cast<std::size_t>(f)]) {
                set_descriptor_field(out, f, py::cast<std::int64_t>(item.second));
                known = true;
            }
        if (!known) throw ValidationError("unknown descriptor field '" + key + "'", key);
    }
    out.check();
    return out;
}

py::dict descriptor_to_dict(const ProblemDescriptor& d) {
    py::dict out;
    for (int f = 0; f < kNumInputFields; ++f) out[kInputFieldNames[static_cast<std::size_t>(f)]] = descriptor_field(d, f);
    out["precision"] = precision_label(d.precision);
    return out;
}

// Opaque Python callable predicate (module.cpp:51-63): evaluated by the
// engine's host hook between positions, under the GIL.
ConstraintPredicate python_predicate(const std::string& name, const std::function<bool(py::dict, py::dict)>& fn) {
    ConstraintPredicate pred;
    pred.name = name;
    pred.fn = [fn](const ProblemDescriptor& d, const ParamMap& partial) {
        py::gil_scoped_acquire gil;
        py::dict params;
        for (const auto& [k, v] : partial) params[py::str(k)] = v;
        return fn(descriptor_to_dict(d), params);
    };
    return pred;
}

py::list beams_to_python(const ModelParams& params, const std::vector<ScoredSequence>& beams) {
    const KernelSpec spec = spec_of(params);
    py::list out;
    for (const ScoredSequence& s : beams) {
        py::dict entry, values;
        for (const auto& [k, v] : decode_params(s.tokens, spec, params.vocab)) values[py::str(k)] = v;
        entry["params"] = values;
        entry["log_prob"] = s.log_prob;
        out.append(entry);
    }
    return out;
}

GemmPrecision precision_of(const std::string& s) {
    if (s == "f16x3") return GemmPrecision::f16x3;
    if (s == "fp32") return GemmPrecision::fp32;
    if (s == "bf16") return GemmPrecision::bf16;
    throw ParameterError("precision must be f16x3, fp32 or bf16");
}

}  // namespace

PYBIND11_MODULE(_kernelseer_b200, m) {
    m.doc() = "B200 constrained beam decode for GPU kernel tuning-parameter prediction";
    py::register_exception<Error>(m, "KernelseerError");

    py::class_<KernelSpec>(m, "KernelSpec")
        .def_readonly("name", &KernelSpec::name)
        .def_property_readonly("params",
                               [](const KernelSpec& s) {
                                   py::list out;
                                   for (const auto& p : s.params) out.append(py::make_tuple(p.name, p.values));
                                   return out;
                               })
        .def("__repr__", [](const KernelSpec& s) {
            return "<KernelSpec " + s.name + " (" + std::to_string(s.num_params()) + " params)>";
        });
    m.def("builtin_specs", [] { return builtin_specs(); });
    m.def("builtin_spec", [](const std::string& n) { return builtin_spec(n); }, py::arg("name"));
    m.def("search_space_size", [](const KernelSpec& s) { return search_space_size(s); }, py::arg("spec"));

    py::class_<Sample>(m, "Sample")
        .def(py::init([](const py::dict& descriptor, const ParamMap& params, const std::string& kernel,
                         const std::string& precision) {
                 Sample s;
                 s.descriptor = descriptor_from_dict(descriptor);
                 s.params = params;
                 s.kernel = kernel;
                 s.precision = precision_from_label(precision);
                 return s;
             }),
             py::arg("descriptor"), py::arg("params"), py::arg("kernel") = "", py::arg("precision") = "fp32")
        .def_property_readonly("descriptor", [](const Sample& s) { return descriptor_to_dict(s.descriptor); })
        .def_readonly("params", &Sample::params)
        .def_readonly("kernel", &Sample::kernel)
        .def_property_readonly("precision", [](const Sample& s) { return precision_label(s.precision); });

    py::class_<PyModel, std::shared_ptr<PyModel>>(m, "ModelParams")
        .def_property_readonly("kernel", [](PyModel& p) { return p.params->kernel; })
        .def_property_readonly("precision", [](PyModel& p) { return precision_label(p.params->precision); })
        .def_property_readonly("variant", [](PyModel& p) { return variant_label(p.params->config.variant); })
        .def_property_readonly("spec", [](PyModel& p) { return spec_of(*p.params); })
        .def("set_engine",
             [](PyModel& p, const py::object& device, const std::string& precision) {
                 std::lock_guard<std::mutex> g(p.mu);
                 p.devices.clear();
                 if (py::isinstance<py::int_>(device)) {
                     p.device = py::cast<int>(device);
                 } else {  // a list of devices (the same GPU may repeat)
                     p.devices = py::cast<std::vector<int>>(device);
                     if (p.devices.empty()) throw ParameterError("empty device list");
                 }
                 p.precision = precision_of(precision);
                 p.predictor.reset();
             },
             py::arg("device") = -1, py::arg("precision") = "f16x3",
             "Select the GPU (-1: every visible GPU, batches sharded across them; or a list of devices) and the gate-GEMM "
             "arithmetic (f16x3 | fp32 | bf16) of the cached engines")
        .def_property_readonly("num_devices", [](PyModel& p) { return p.pred().num_devices(); })
        .def("__repr__", [](PyModel& p) {
            return "<ModelParams " + variant_label(p.params->config.variant) + " for " + p.params->kernel + ">";
        });
    m.def("load_checkpoint",
          [](const std::string& path) {
              auto pm = std::make_shared<PyModel>();
              pm->params = std::make_shared<ModelParams>(load_checkpoint(path));
              return pm;
          },
          py::arg("path"));

    py::class_<ConstraintPredicate>(m, "ConstraintPredicate")
        .def_readonly("name", &ConstraintPredicate::name)
        .def_property_readonly("device_evaluable", [](const ConstraintPredicate& p) { return (bool)p.program; });
    m.def("membership_predicate", &membership_predicate, py::arg("spec"));
    m.def("resource_budget_predicate",
          [](const std::map<std::string, double>& w, double budget, const std::string& name) {
              return resource_budget_predicate(w, budget, name);
          },
          py::arg("weights"), py::arg("budget"), py::arg("name") = "resource_budget");
    m.def("product_limit_predicate", &product_limit_predicate, py::arg("params"), py::arg("scale"),
          py::arg("limit"), py::arg("name") = "product_limit",
          "scale * prod(assigned values) <= limit (workgroup size / LDS bytes); device-evaluated");
    m.def("divisibility_predicate", &divisibility_predicate, py::arg("param_field"),
          py::arg("name") = "divisibility",
          "each listed parameter value divides descriptor field (0..6 = n,c,h,w,k,y,x); device-evaluated");
    m.def("predicate", &python_predicate, py::arg("name"), py::arg("fn"),
          "Wrap a python callable (descriptor_dict, partial_params_dict) -> bool (host-evaluated)");

    m.def("validate",
          [](const KernelSpec& spec, const py::dict& descriptor, const ParamMap& params,
             const std::vector<ConstraintPredicate>& predicates) -> py::object {
              const auto v = validate_sequence(spec, descriptor_from_dict(descriptor), params, predicates);
              if (!v) return py::none();
              py::dict out;
              out["predicate"] = v->predicate;
              out["params"] = v->params;
              return out;
          },
          py::arg("spec"), py::arg("descriptor"), py::arg("params"), py::arg("predicates"));

    m.def("predict",
          [](std::shared_ptr<PyModel> pm, const py::dict& descriptor, int beam_width,
             const std::vector<ConstraintPredicate>& predicates, bool snap) {
              const ProblemDescriptor d = descriptor_from_dict(descriptor);
              const TokenSequence input = encode_problem(d, pm->params->vocab, snap);
              const SequencePredictor& pred = pm->pred();
              std::vector<ScoredSequence> beams;
              {
                  py::gil_scoped_release nogil;
                  beams = predicates.empty() ? beam_search(pred, input, beam_width)
                                             : constrained_beam_search(pred, input, beam_width, predicates, d);
              }
              return beams_to_python(*pm->params, beams);
          },
          py::arg("params"), py::arg("descriptor"), py::arg("beam_width") = 1,
          py::arg("predicates") = std::vector<ConstraintPredicate>{}, py::arg("snap") = false);

    m.def("greedy_predict",
          [](std::shared_ptr<PyModel> pm, const py::dict& descriptor, bool snap) {
              const ProblemDescriptor d = descriptor_from_dict(descriptor);
              const TokenSequence input = encode_problem(d, pm->params->vocab, snap);
              const SequencePredictor& pred = pm->pred();
              TokenSequence out;
              {
                  py::gil_scoped_release nogil;
                  out = greedy_decode(pred, input);
              }
              py::dict values;
              for (const auto& [k, v] : decode_params(out, spec_of(*pm->params), pm->params->vocab))
                  values[py::str(k)] = v;
              return values;
          },
          py::arg("params"), py::arg("descriptor"), py::arg("snap") = false);

    m.def("predict_batch",
          [](std::shared_ptr<PyModel> pm, const std::vector<py::dict>& descriptors, int beam_width,
             const std::vector<ConstraintPredicate>& predicates, bool snap) {
              std::vector<ProblemDescriptor> ds;
              std::vector<TokenSequence> ins;
              for (const auto& dd : descriptors) {
                  ds.push_back(descriptor_from_dict(dd));
                  ins.push_back(encode_problem(ds.back(), pm->params->vocab, snap));
              }
              const SequencePredictor& pred = pm->pred();
              BatchResult r;
              {
                  py::gil_scoped_release nogil;
                  r = beam_search_batch(pred, ins, ds, beam_width, predicates);
              }
              py::list out;
              for (std::size_t i = 0; i < ins.size(); ++i) {
                  if (r.exhausted[i].exhausted) {
                      py::dict e;
                      e["exhausted"] = true;
                      e["predicate"] = r.exhausted[i].predicate;
                      e["step"] = r.exhausted[i].step;
                      out.append(e);
                  } else {
                      out.append(beams_to_python(*pm->params, r.beams[i]));
                  }
              }
              return out;
          },
          py::arg("params"), py::arg("descriptors"), py::arg("beam_width") = 1,
          py::arg("predicates") = std::vector<ConstraintPredicate>{}, py::arg("snap") = false,
          "Batched predict: one entry per descriptor (a beam list, or an exhaustion record)");

    // ------------------------------------------------------------ stepping facade
    // (models.hpp:65-103; the reference's pybind module does not bind these --
    // B200 additions for the teacher-forced scorer and the stepping API)
    m.def("encode_problem",
          [](std::shared_ptr<PyModel> pm, const py::dict& descriptor, bool snap) {
              return encode_problem(descriptor_from_dict(descriptor), pm->params->vocab, snap).ids;
          },
          py::arg("params"), py::arg("descriptor"), py::arg("snap") = false,
          "encode_problem (encoding.cpp:87-113): 7 input token ids; ValidationError naming the field");
    m.def("model_forward",
          [](std::shared_ptr<PyModel> pm, const std::vector<std::vector<int>>& inputs,
             const std::optional<std::vector<std::vector<int>>>& teachers) {
              std::vector<TokenSequence> ins;
              for (const auto& t : inputs) {
                  TokenSequence s;
                  s.ids = t;
                  ins.push_back(std::move(s));
              }
              const SequencePredictor& pred = pm->pred();
              std::vector<double> scores;
              std::vector<std::vector<nn::Tensor>> d;
              std::vector<std::vector<int>> tch = teachers ? *teachers : std::vector<std::vector<int>>{};
              {
                  py::gil_scoped_release nogil;
                  d = model_forward_batch(pred, ins, tch, &scores);
              }
              py::list dists;
              for (const auto& row : d) {
                  py::list r;
                  for (const auto& t : row) r.append(t.values());
                  dists.append(r);
              }
              return py::make_tuple(dists, scores);
          },
          py::arg("params"), py::arg("inputs"), py::arg("teachers") = py::none(),
          "model_forward (models.cpp:495-514) over many input token sequences in one device pass: "
          "(per input, per position distributions; per input sequence score sum log max(p, 1e-300))");

    py::class_<EncodedInput>(m, "EncodedInput")
        .def_property_readonly("input", [](const EncodedInput& e) { return e.input.ids; });
    py::class_<DecoderState>(m, "DecoderState")
        .def_readonly("position", &DecoderState::position)
        .def_readonly("fed", &DecoderState::fed);
    struct PyPredictor {
        std::shared_ptr<PyModel> pm;
    };
    py::class_<PyPredictor>(m, "SequencePredictor")
        .def(py::init([](std::shared_ptr<PyModel> pm) { return PyPredictor{pm}; }), py::arg("params"))
        .def("num_positions", [](PyPredictor& p) { return p.pm->pred().num_positions(); })
        .def("vocab_size", [](PyPredictor& p, int pos) { return p.pm->pred().vocab_size(pos); }, py::arg("position"))
        .def("encode",
             [](PyPredictor& p, const std::vector<int>& ids) {
                 TokenSequence s;
                 s.ids = ids;
                 return p.pm->pred().encode(s);
             },
             py::arg("input"))
        .def("initial_state", [](PyPredictor& p, const EncodedInput& e) { return p.pm->pred().initial_state(e); },
             py::arg("enc"))
        .def("step",
             [](PyPredictor& p, const EncodedInput& e, DecoderState& st, int prev) {
                 const SequencePredictor& pred = p.pm->pred();
                 nn::Tensor t;
                 {
                     py::gil_scoped_release nogil;
                     t = pred.step(e, st, prev);
                 }
                 return t.values();
             },
             py::arg("enc"), py::arg("state"), py::arg("prev_token"));

    m.def("device_count", [] { return ks_device_count(); }, "visible CUDA devices");
    m.def("synthetic_descriptors",
          [](std::shared_ptr<PyModel> pm, std::int64_t count, std::uint64_t seed, std::int64_t start) {
              const auto ds = synthetic_descriptors(*pm->params, count, seed, start);
              py::array_t<std::int64_t> out({(py::ssize_t)count, (py::ssize_t)7});
              auto w = out.mutable_unchecked<2>();
              for (std::int64_t i = 0; i < count; ++i)
                  for (int f = 0; f < 7; ++f) w(i, f) = descriptor_field(ds[(std::size_t)i], f);
              return out;
          },
          py::arg("params"), py::arg("count"), py::arg("seed") = 2404, py::arg("start") = 0,
          "Workload configs start..start+count-1 (count x 7: n,c,h,w,k,y,x), config i from Rng::derive(seed, i)");

    m.def("topk_metrics",
          [](std::shared_ptr<PyModel> pm, const std::vector<Sample>& test, const std::vector<int>& k_values,
             const std::vector<ConstraintPredicate>& predicates, int threads) {
              std::vector<EvalReport> reports;
              const SequencePredictor& pred = pm->pred();
              {
                  py::gil_scoped_release nogil;
                  reports = topk_metrics(pred, test, k_values, predicates, threads);
              }
              py::list out;
              for (const EvalReport& r : reports) {
                  py::dict d;
                  d["beam_width"] = r.beam_width;
                  d["constrained"] = r.constrained;
                  d["samples"] = r.sample_count;
                  d["average_accuracy"] = r.average_accuracy;
                  d["perfect_prediction"] = r.perfect_prediction;
                  d["per_param_accuracy"] = r.per_param_accuracy;
                  out.append(d);
              }
              return out;
          },
          py::arg("params"), py::arg("test"), py::arg("k_values"),
          py::arg("predicates") = std::vector<ConstraintPredicate>{}, py::arg("threads") = 1);
    // ------------------------------------------------------------ training
    // (bindings/module.cpp:183-256): same class / kwargs / defaults; the batches
    // run on the GPU (enc-dec / attn / attn-2).
    py::class_<ModelConfig>(m, "ModelConfig")
        .def(py::init([](const std::string& variant, int encoder_state_size, int pre_attention_size,
                         int post_attention_size, int attention_dense_nodes,
                         const std::vector<std::tuple<int, int, int>>& conv_layers, int decoder_cell_size,
                         double dropout, double recurrent_dropout) {
                 ModelConfig c;
                 c.variant = variant_from_label(variant);
                 c.encoder_state_size = encoder_state_size;
                 c.pre_attention_size = pre_attention_size;
                 c.post_attention_size = post_attention_size;
                 c.attention_dense_nodes = attention_dense_nodes;
                 c.conv_layers.clear();
                 for (const auto& [f, k, st] : conv_layers) c.conv_layers.push_back({f, k, st});
                 c.decoder_cell_size = decoder_cell_size;
                 c.dropout = dropout;
                 c.recurrent_dropout = recurrent_dropout;
                 if (encoder_state_size < 1 || pre_attention_size < 1 || post_attention_size < 1 ||
                     attention_dense_nodes < 1 || decoder_cell_size < 1)
                     throw ParameterError("model sizes must be >= 1");
                 if (dropout < 0.0 || dropout >= 1.0 || recurrent_dropout < 0.0 || recurrent_dropout >= 1.0)
                     throw ParameterError("dropout rates must be in [0,1)");
                 return c;
             }),
             py::arg("variant") = "hybrid-2", py::arg("encoder_state_size") = 256, py::arg("pre_attention_size") = 256,
             py::arg("post_attention_size") = 512, py::arg("attention_dense_nodes") = 2,
             py::arg("conv_layers") = std::vector<std::tuple<int, int, int>>{{64, 3, 1}, {32, 3, 1}},
             py::arg("decoder_cell_size") = 256, py::arg("dropout") = 0.2, py::arg("recurrent_dropout") = 0.2)
        .def_property_readonly("variant", [](const ModelConfig& c) { return variant_label(c.variant); });

    m.def("train",
          [](const ModelConfig& config, const KernelSpec& spec, const std::vector<Sample>& train_set,
             const std::vector<Sample>& test_set, int epochs, int batch_size, std::uint64_t seed, int threads,
             double learning_rate, int device) {
              std::vector<Sample> all = train_set;
              all.insert(all.end(), test_set.begin(), test_set.end());
              const Vocabulary vocab = build_vocab(spec, all);
              const Precision precision = train_set.empty() ? Precision::full : train_set[0].precision;
              TrainOptions o;
              o.epochs = epochs;
              o.batch_size = batch_size;
              o.seed = seed;
              o.threads = threads;
              o.learning_rate = learning_rate;
              TrainResult r;
              {
                  py::gil_scoped_release release;
                  r = train_model(config, spec, vocab, precision, train_set, test_set, o, {}, device);
              }
              py::list log;
              for (const EpochStats& e : r.log) {
                  py::dict row;
                  row["epoch"] = e.epoch;
                  row["train_loss"] = e.train_loss;
                  row["train_avg_acc"] = e.train_accuracy;
                  row["test_loss"] = e.test_loss;
                  row["test_avg_acc"] = e.test_accuracy;
                  log.append(row);
              }
              auto pm = std::make_shared<PyModel>();
              pm->params = std::make_shared<ModelParams>(std::move(r.params));
              pm->device = device;
              return py::make_tuple(pm, log);
          },
          py::arg("config"), py::arg("spec"), py::arg("train_set"), py::arg("test_set"), py::arg("epochs") = 30,
          py::arg("batch_size") = 32, py::arg("seed") = 1, py::arg("threads") = 1, py::arg("learning_rate") = 1e-3,
          py::arg("device") = 0);

    m.def("init_model",
          [](const ModelConfig& config, const KernelSpec& spec, const std::vector<Sample>& samples, std::uint64_t seed) {
              auto pm = std::make_shared<PyModel>();
              pm->params = std::make_shared<ModelParams>(
                  init_model(config, spec, build_vocab(spec, samples),
                             samples.empty() ? Precision::full : samples[0].precision, seed));
              return pm;
          },
          py::arg("config"), py::arg("spec"), py::arg("samples"), py::arg("seed") = 1,
          "init_model (models.cpp:178-259) over build_vocab(spec, samples)");
    m.def("save_checkpoint", [](const std::shared_ptr<PyModel>& p, const std::string& path) { save_checkpoint(*p->params, path); },
          py::arg("params"), py::arg("path"));
}
