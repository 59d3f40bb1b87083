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

There is no CPU fallback: importing without the built extension raises.
"""
__version__ = "0.1.0"

from ._kernelseer_b200 import (  # noqa: F401
    ConstraintPredicate,
    KernelSpec,
    KernelseerError,
    ModelConfig,
    ModelParams,
    Sample,
    builtin_spec,
    builtin_specs,
    divisibility_predicate,
    greedy_predict,
    init_model,
    load_checkpoint,
    membership_predicate,
    predict,
    predict_batch,
    predicate,
    product_limit_predicate,
    resource_budget_predicate,
    save_checkpoint,
    search_space_size,
    topk_metrics,
    train,
    validate,
)
