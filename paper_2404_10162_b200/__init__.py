"""B200-native constrained beam-decode engine for the kernel-tuning-parameter
translator of arXiv 2404.10162 (reference: kernelseer).

The hot path (LSTM encoder -> attention decoder -> constrained beam search)
runs as hand-written sm_100a CUDA behind the C-ABI in include/ks_b200.h.  This
package re-exports the reference binding's names (proj/bindings/module.cpp)
for the decode path, so `import paper_2404_10162_b200 as ks` stands in for
`import kernelseer as ks`:

    params = ks.load_checkpoint(path)
    ks.predict(params, {"n": 32, "c": 256, ...}, beam_width=5,
               predicates=[ks.membership_predicate(params.spec),
                           ks.resource_budget_predicate({...}, 60.0)])

The binding (_kernelseer_b200 -> libkernelseer_b200.so -> libks_b200.so) is
loaded on first use of any of these names (PEP 562), so pure-Python helpers
(specs, synth, parallel) import without mapping the engine -- the reference
arm of bench.py relies on that.  There is no CPU fallback: using the API
without the built extension raises ImportError.
"""
__version__ = "0.1.0"

_API = (
    "ConstraintPredicate", "KernelSpec", "KernelseerError", "ModelConfig", "ModelParams", "Sample",
    "SequencePredictor", "EncodedInput", "DecoderState",
    "builtin_spec", "builtin_specs", "divisibility_predicate", "greedy_predict", "init_model",
    "load_checkpoint", "membership_predicate", "model_forward", "predict", "predict_batch", "predicate",
    "product_limit_predicate", "resource_budget_predicate", "save_checkpoint", "search_space_size",
    "synthetic_descriptors", "topk_metrics", "train", "validate", "encode_problem", "device_count",
)


def __getattr__(name):
    if name in _API:
        from . import _kernelseer_b200 as _m

        try:
            v = getattr(_m, name)
        except AttributeError:
            raise AttributeError(f"module {__name__!r} has no attribute {name!r}") from None
        globals()[name] = v
        return v
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")


def __dir__():
    return sorted(list(globals()) + list(_API))
