"""Diagnose the reference's gradient check (criterion 01) on the drop-in:
repeatability of loss_and_grad and the worst finite-difference coordinate.
Run from baseline/_ref/ref_tests with tools/kgdist_alias on PYTHONPATH."""
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
from test_model import _setup, _flat_arrays  # noqa: E402
from kgdist.model import loss_and_grad, MODE_EMBEDDING  # noqa: E402

for seed in range(5):
    _, config, params, _, batch, cg, table, ids = _setup(num_entities=12 + 3 * seed, num_relations=2, num_edges=30,
                                                         seed=seed, dims=(3, 4, 2))
    runs = [loss_and_grad(params, config, batch, cg, params.entity_embed, ids) for _ in range(4)]
    l0 = [r[0] for r in runs]
    same_loss = all(x == l0[0] for x in l0)
    g0 = [np.concatenate([g.ravel() for g in r[1].dense_blocks()]) for r in runs]
    same_grad = all(np.array_equal(g0[0], g) for g in g0)
    loss, grads = runs[0]
    analytic = [g.copy() for g in grads.dense_blocks()]
    dense_embed = np.zeros_like(params.entity_embed)
    dense_embed[grads.embed_ids] += grads.embed_rows
    analytic.append(dense_embed)
    worst, where = 0.0, None
    names = ["bases%d" % i for i in range(len(params.bases))] + ["coeffs%d" % i for i in range(len(params.coeffs))] + \
        ["decoder", "embed"]
    for name, arr, ana in zip(names, _flat_arrays(params, config), analytic):
        flat, aflat = arr.reshape(-1), ana.reshape(-1)
        for i in range(flat.size):
            orig = flat[i]
            flat[i] = orig + 1e-5
            lp = loss_and_grad(params, config, batch, cg, params.entity_embed, ids)[0]
            flat[i] = orig - 1e-5
            lm = loss_and_grad(params, config, batch, cg, params.entity_embed, ids)[0]
            flat[i] = orig
            fd = (lp - lm) / 2e-5
            err = abs(fd - aflat[i]) / max(abs(fd), abs(aflat[i]), 1e-8)
            if err > worst:
                worst, where = err, (name, i, fd, aflat[i])
    print(f"seed {seed}: loss repeat-equal {same_loss} grad repeat-equal {same_grad} loss {l0[0]!r} "
          f"worst {worst:.2e} at {where}", flush=True)
