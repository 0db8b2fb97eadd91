"""GPU parity of the standalone LAYERNORM and DROPOUT layer kinds (include/tgp.h; PAPER.md P:122 a
partition is any sequence of layers; P:105 / P:212 the recompute regenerates the dropout mask from the
restored RNG state) against the fp64 oracle (oracle/model.py, pinned in tests/test_oracle_model.py
against torch autograd and finite differences): fp32 mode at 1e-4, bf16 mode at 2e-2 normwise
(reading Z15); every checkpoint mode bitwise equal (F' == F, reading Z21)."""
import numpy as np
import pytest

from synth import configs as C

from _gpu import compare, gpu_step, make_case, oracle_step

pytestmark = pytest.mark.gpu


def _case(layers, B, m, n, ckpt, dtype, seed=21, steps=1):
    x, t, params = make_case(layers, B, seed, dtype)
    g, P = gpu_step(layers, params, x, t, m=m, n=n, ckpt=ckpt, dtype=dtype, lr=0.05, seed=seed, steps=steps)
    P.close()
    return x, t, params, g


@pytest.mark.parametrize("dtype,tol,d", [("fp32", 1e-4, 128), ("bf16", 2e-2, 512)])
def test_ln_dropout_stack_matches_oracle(dtype, tol, d):
    layers = C.ln_mlp(3, d, dropout=0.1)
    x, t, params, g = _case(layers, 48, 3, 2, "except_last", dtype)
    ref = oracle_step(layers, params, x, t, lr=0.05, m=3, seed=21, step=0)
    errs, bad = compare(g, ref, params, tol, 0.05)
    assert not bad, bad


def test_resmlp_around_layernorm_and_dropout_bf16():
    # RESMLP blocks next to the new kinds: the RESMLP backward must form its own bf16 dY operand
    # when the layer above is not a RESMLP (no LN-backward fusion)
    L = [C.layer("resmlp", 512, 512, d_hidden=1024, act="gelu"), C.layer("layernorm", 512, 512),
         C.layer("dropout", 512, 512, dropout=0.2), C.layer("resmlp", 512, 512, d_hidden=512, act="gelu"),
         C.layer("layernorm", 512, 512), C.layer("linear", 512, 512)]
    x, t, params, g = _case(L, 64, 4, 2, "always", "bf16")
    ref = oracle_step(L, params, x, t, lr=0.05, m=4, seed=21, step=0)
    errs, bad = compare(g, ref, params, 2e-2, 0.05)
    assert not bad, bad


def test_ln_dropout_checkpoint_modes_bitwise():
    layers = C.ln_mlp(2, 256, dropout=0.3)
    res = {}
    for mode in ("always", "except_last", "never"):
        x, t, params, g = _case(layers, 32, 4, 2, mode, "bf16", steps=2)
        res[mode] = g
    for mode in ("except_last", "never"):
        for a, b in zip(res[mode], res["always"]):
            assert a["loss"] == b["loss"]
            assert np.array_equal(a["dx"], b["dx"])
            for ga, gb in zip(a["grads"], b["grads"]):
                assert np.array_equal(ga, gb)
