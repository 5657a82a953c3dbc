"""Loss-curve fixture: the REAL reference ``run_training`` (trainer.py:440-537) on the
copy task, recorded every step (VERDICT r1 "Next round" #8).

Run in the build container (imports ``int8flow`` from /root/reference unmodified):

    python tests/golden/make_losscurve.py

Freezes the training config, the model's initial FP32 parameters (the same seeded
draws ``run_training`` makes), every step's training batch and the records
(train loss, validation loss, gradient norm per step) into
``tests/golden/losscurve.npz``.  The GPU test trains the same model from the same
parameters on the same batches and compares the curves.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

STEPS = 60


def main():
    sys.path.insert(0, REF_SRC)
    from int8flow import trainer

    cfg = trainer.TrainConfig(layers=2, c_model=64, heads=4, mlp_ratio=4, steps=STEPS, lr=2e-3, weight_decay=0.1,
                              seed=5, batch_size=8, eval_every=1, eval_batches=1)
    task = trainer.CopySequence(vocab=16, length=32)
    records = trainer.run_training(cfg, task)
    assert len(records) == STEPS and not any(r.diverged for r in records)
    sampler = trainer.make_sampler(task)
    model = trainer.ToyModel(cfg, sampler.vocab)  # same seeded draws as inside run_training
    out = {"cfg": np.array([cfg.layers, cfg.c_model, cfg.heads, cfg.hidden, sampler.vocab, cfg.batch_size]),
           "lr": np.float64(cfg.lr), "weight_decay": np.float64(cfg.weight_decay),
           "decay_keys": np.array(sorted(model.decay_keys))}
    for k, v in model.params.items():
        out["p_" + k] = v.copy()
    xs, ys, ms = [], [], []
    for step in range(STEPS):
        x, y, mask = sampler.batch(cfg.seed, step, cfg.batch_size, cfg.block, False)
        xs.append(x)
        ys.append(y)
        ms.append(mask)
    vx, vy, vm = sampler.batch(cfg.seed, 0, cfg.batch_size, cfg.block, True)
    out.update(x=np.stack(xs), y=np.stack(ys), mask=np.stack(ms), val_x=vx, val_y=vy, val_mask=vm,
               train_loss=np.array([r.train_loss for r in records]),
               val_loss=np.array([r.val_loss for r in records]),
               grad_norm=np.array([r.grad_norm for r in records]))
    np.savez_compressed(os.path.join(HERE, "losscurve.npz"), **out)
    print("losscurve.npz written: train loss", records[0].train_loss, "->", records[-1].train_loss)


if __name__ == "__main__":
    main()
