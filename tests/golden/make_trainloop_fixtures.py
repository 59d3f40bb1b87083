"""Fixtures for the drop-in `train` API (reference bindings/module.cpp:222-256,
train_model models.cpp:862-969), made with the UNMODIFIED reference's own
pybind module (oracle/_ref/_kernelseer*.so, compiled from
/root/reference/proj by `make -C oracle ref`):

* trainloop_data.json   a ConvAsm1x1U synthetic dataset (generate_synthetic,
                        split) as plain descriptors / parameter maps;
* trainloop_init.ckpt   init_model of the fixture config over the first 64 / 16
                        samples -- ks.train with learning_rate 0 leaves the
                        initialisation unchanged (Adam's step is lr * ...);
* trainloop_ref.ckpt    the reference's ks.train, 2 epochs, dropout 0.2 / 0.2;
  trainloop_log.json    its per-epoch log.

    make -C oracle ref && python tests/golden/make_trainloop_fixtures.py
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
CONFIG = dict(variant="attn", pre_attention_size=16, post_attention_size=32, attention_dense_nodes=2,
              dropout=0.2, recurrent_dropout=0.2)
TRAIN = dict(epochs=2, batch_size=32, seed=3, learning_rate=3e-3)
INIT_N = (64, 16)


def main():
    sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
    import _kernelseer as ks

    spec = ks.builtin_spec("ConvAsm1x1U")
    ds = ks.generate_synthetic(spec, 800, seed=7, difficulty="moderate")
    train, test = ks.split(ds, 0.25, seed=7)
    rows = lambda ss: [{"descriptor": {k: v for k, v in s.descriptor.items() if k != "precision"},
                        "params": dict(s.params)} for s in ss]
    data = {"kernel": "ConvAsm1x1U", "train": rows(train.samples), "test": rows(test.samples)}
    with open(os.path.join(HERE, "trainloop_data.json"), "w") as f:
        json.dump(data, f)
    cfg = ks.ModelConfig(**CONFIG)
    p0, _ = ks.train(cfg, spec, train.samples[:INIT_N[0]], test.samples[:INIT_N[1]], epochs=1, batch_size=64,
                     seed=TRAIN["seed"], threads=1, learning_rate=0.0)
    ks.save_checkpoint(p0, os.path.join(HERE, "trainloop_init.ckpt"))
    p, log = ks.train(cfg, spec, train.samples, test.samples, threads=4, **TRAIN)
    ks.save_checkpoint(p, os.path.join(HERE, "trainloop_ref.ckpt"))
    with open(os.path.join(HERE, "trainloop_log.json"), "w") as f:
        json.dump(log, f, indent=1)
    print(len(train.samples), len(test.samples), log)


if __name__ == "__main__":
    main()
