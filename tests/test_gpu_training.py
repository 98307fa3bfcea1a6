"""One encrypted training step (Alg. 6) on the
GPU: every intermediate (pre-activations, activations, error signs, gradient
signs) and the updated weights decrypt to the cleartext Alg. 6 of
oracle.gadgets.train_step on every element."""
import json
import os
import time

import numpy as np
import pytest
import torch

from oracle import gadgets as G
from synth import get_params, lwe_randomness, streams

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    return torch.device("cuda:0")


def run_step(dims, batch, seed, dev, small_n):
    from paper_2504_17785_b200 import training as TR, workload as wl
    PA = get_params("A_SMALLN" if small_n else "A")
    PB = get_params("B_SMALLN" if small_n else "B")
    t0 = time.perf_counter()
    ctx = TR.make_context(PA, PB, seed, dev)
    torch.cuda.synchronize()
    t_keys = time.perf_counter() - t0
    rng = streams(seed)["messages"]
    A0 = rng.integers(-8, 8, size=(batch, dims[0]))
    Ws = [rng.integers(-8, 8, size=(dims[l + 1], dims[l])) for l in range(len(dims) - 1)]
    Y = np.zeros((batch, dims[-1]), dtype=np.int64)
    Y[np.arange(batch), rng.integers(0, dims[-1], size=batch)] = 1
    key = ctx.ka["big_key"]
    enc = lambda x, s: wl.encrypt(PA, np.asarray(x).reshape(-1), lwe_randomness(PA, np.asarray(x).size, s), key,  # noqa: E731
                                  dev).reshape(*np.asarray(x).shape, -1)
    A0c, Yc = enc(A0, seed + 10), enc(Y, seed + 11)
    Wc = [enc(W, seed + 20 + l) for l, W in enumerate(Ws)]
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    newW, it = ctx.train_step(A0c, Yc, Wc, keep=True)
    torch.cuda.synchronize()
    t_step = time.perf_counter() - t1
    refW, ref = G.train_step(A0, Y, Ws)
    return ctx, newW, it, refW, ref, {"keygen_s": t_keys, "step_s": t_step}


def check(ctx, newW, it, refW, ref):
    L = len(refW)
    for l in range(L):
        got = ctx.decrypt(it["pre"][l]).reshape(ref["pre"][l].shape)
        assert np.array_equal(got, ref["pre"][l]), f"pre-activation {l}"
        got = ctx.decrypt(it["acts"][l + 1]).reshape(ref["acts"][l + 1].shape)
        assert np.array_equal(got, ref["acts"][l + 1]), f"activation {l}"
        got = ctx.decrypt(it["grads"][l]).reshape(ref["grads"][l].shape)
        assert np.array_equal(got, ref["grads"][l]), f"gradient sign {l}"
        got = ctx.decrypt(newW[l]).reshape(refW[l].shape)
        assert np.array_equal(got, refW[l]), f"updated weights {l}"
    for e_got, e_ref in zip(it["errs"], ref["errs"]):
        assert np.array_equal(ctx.decrypt(e_got).reshape(e_ref.shape), e_ref), "error signs"


def test_train_step_tiny_small_n(dev):
    """MLP 6-3-2, batch 4, small-n parameter sets (fast)."""
    check(*run_step([6, 3, 2], 4, 91, dev, small_n=True)[:5])


def test_train_steps_chain(dev):
    """Two consecutive steps (R26): the second step starts from the encrypted
    weights the first produced (fresh PBS outputs) and a new batch, and still
    decrypts to the cleartext Alg. 6 everywhere."""
    from paper_2504_17785_b200 import workload as wl
    ctx, newW, it, refW, ref, _ = run_step([6, 3, 2], 4, 93, dev, small_n=True)
    check(ctx, newW, it, refW, ref)
    PA = ctx.PA
    rng = streams(94)["messages"]
    A0 = rng.integers(-8, 8, size=(4, 6))
    Y = np.zeros((4, 2), dtype=np.int64)
    Y[np.arange(4), rng.integers(0, 2, size=4)] = 1
    key = ctx.ka["big_key"]
    enc = lambda x, s: wl.encrypt(PA, np.asarray(x).reshape(-1), lwe_randomness(PA, np.asarray(x).size, s), key,  # noqa: E731
                                  dev).reshape(*np.asarray(x).shape, -1)
    newW2, it2 = ctx.train_step(enc(A0, 95), enc(Y, 96), newW, keep=True)
    refW2, ref2 = G.train_step(A0, Y, refW)
    check(ctx, newW2, it2, refW2, ref2)


def test_train_step_paper_shaped_mlp(dev):
    """The paper's smallest MLP shape (28-8-2, batch 8) at the full
    parameter sets (n = 742 / 1024)."""
    ctx, newW, it, refW, ref, rep = run_step([28, 8, 2], 8, 92, dev, small_n=False)
    check(ctx, newW, it, refW, ref)
    rep["stage_s"] = it["times"]
    rep.update({"workload": "Alg. 6 training step, MLP 28-8-2, batch 8, set A + set-B Shift2MSBs stage",
                "weights_changed": [int((r != W0).sum()) for r, W0 in zip(refW, ref["W_in"])]})
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/train_step.json", "w") as f:
        json.dump(rep, f)
    print(json.dumps(rep))
