"""GPU parity tests: the CUDA pipeline (through the C ABI) vs the fp64 oracle on the same seeded
inputs.  Bars (BASELINE.json north_star, reading Z15): loss, y, dx, every gradient and every
delta-theta within normwise 1e-4 in fp32 mode and 2e-2 in bf16 mode.  Multi-partition runs place
all partitions on cuda:0 (separate streams, same-device copies) -- the multi-GPU transport is the
same code path with peer pointers."""
import numpy as np
import pytest

from synth import configs as C

from _gpu import compare, gpu_step, make_case, oracle_step

pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-4, "bf16": 2e-2}


def _check(layers, B, m, n, ckpt, dtype, lr=0.1, balance=None, seed=7, options=None):
    x, t, params = make_case(layers, B, seed, dtype)
    ref = oracle_step(layers, params, x, t, lr=lr, m=m, seed=seed, step=0)
    gpu, P = gpu_step(layers, params, x, t, m=m, n=n, ckpt=ckpt, dtype=dtype, lr=lr, balance=balance, seed=seed,
                      options=options)
    errs, bad = compare(gpu, ref, params, TOL[dtype], lr)
    assert not bad, f"errors above {TOL[dtype]}: {bad}"
    return gpu, ref, errs, P


def test_c1_fp32_parity():
    cfg = C.C1()
    gpu, ref, errs, P = _check(cfg.layers, cfg.batch, cfg.m, cfg.n, cfg.checkpoint, cfg.dtype, cfg.lr, cfg.balance)
    # the runtime issued exactly the oracle's schedule (bit-exact integer records, O5)
    from oracle.schedule import records
    want = records(cfg.m, cfg.n, cfg.checkpoint)
    assert np.array_equal(gpu["log"], want)


@pytest.mark.parametrize("mode", ["always", "except_last", "never"])
@pytest.mark.parametrize("m,n", [(1, 1), (4, 2), (3, 4)])
def test_mlp_fp32_modes(mode, m, n):
    layers = C.mlp_chain(8, 64, act="gelu")
    layers[3]["dropout"] = 0.2
    _check(layers, 12, m, n, mode, "fp32", balance=[8 // n + (1 if j < 8 % n else 0) for j in range(n)])


def test_resmlp_fp32_parity():
    layers = C.resmlp_stack(4, 128, hidden=256, dropout=0.1)
    _check(layers, 32, 4, 2, "except_last", "fp32")


@pytest.mark.parametrize("stream", [0, 1])
def test_c2_small_bf16_parity(stream):
    # stream = 1: the persistent weight-streaming task kernel (n = 2 partitions on one device, both
    # fit co-resident at d = 512); stream = 0: the per-layer kernel path
    layers = C.resmlp_stack(8, 512)
    _check(layers, 64, 4, 2, "except_last", "bf16", lr=0.05, options={"stream": stream})


def test_c2_small_bf16_dropout_always():
    layers = C.resmlp_stack(4, 256, hidden=512, dropout=0.1)
    _check(layers, 64, 4, 4, "always", "bf16", lr=0.05)


def test_c4_small_bf16_skip_routes():
    # U-MLP with 4 long skip routes crossing partitions (portals: one direct copy per micro-batch)
    layers = C.umlp(d=256)
    bal = [2, 3, 3, 3, 3, 3, 3, 3]
    gpu, ref, errs, P = _check(layers, 32, 4, 8, "except_last", "bf16", lr=0.05, balance=bal)
    log = gpu["log"]
    from oracle.schedule import SKIP_F, records, route_partitions
    want = records(4, 8, "except_last", route_partitions(layers, bal))
    assert np.array_equal(log, want)
    assert int((log[:, 2] == SKIP_F).sum()) == 4 * 4


def test_c4_small_fp32_skip_routes_same_partition():
    layers = C.umlp(d=64, levels=2, blocks_per_level=1, mid_blocks=1)
    _check(layers, 16, 4, 2, "never", "fp32", balance=[3, len(layers) - 3])


def test_bn_fp32_parity():
    cfg = C.BN()
    gpu, ref, errs, P = _check(cfg.layers, cfg.batch, cfg.m, cfg.n, cfg.checkpoint, cfg.dtype, cfg.lr, cfg.balance)
    k = 0
    for li, L in enumerate(cfg.layers):
        if L["kind"] == "batchnorm":
            rm, rv = P.bn_running(li, L["d_in"])
            em, ev = ref["bn"][k]
            k += 1
            assert np.max(np.abs(rm - em)) <= 1e-4 * max(1.0, np.max(np.abs(em)))
            assert np.max(np.abs(rv - ev)) <= 1e-4 * max(1.0, np.max(np.abs(ev)))


def test_checkpoint_modes_bitwise_identical_bf16():
    # F' reproduces F bit-exactly (referential transparency P:122 fn, reading Z21): the gradients of
    # always / except_last / never must be BITWISE equal on the GPU, dropout included.
    layers = C.resmlp_stack(4, 256, dropout=0.1)
    x, t, params = make_case(layers, 64, 3, "bf16")
    res = {}
    for mode in ("always", "except_last", "never"):
        g, P = gpu_step(layers, params, x, t, m=4, n=2, ckpt=mode, dtype="bf16", lr=0.05, seed=3)
        res[mode] = g
        P.close()
    for mode in ("except_last", "never"):
        assert res[mode]["loss"] == res["always"]["loss"]
        for a, b in zip(res[mode]["grads"], res["always"]["grads"]):
            assert np.array_equal(a, b)


def test_graphs_and_eager_bitwise_identical():
    layers = C.resmlp_stack(3, 256)
    x, t, params = make_case(layers, 32, 5, "bf16")
    g1, P1 = gpu_step(layers, params, x, t, m=2, n=3, ckpt="except_last", dtype="bf16", lr=0.05,
                      options={"graphs": 0, "pdl": 0})
    g2, P2 = gpu_step(layers, params, x, t, m=2, n=3, ckpt="except_last", dtype="bf16", lr=0.05)
    for a, b in zip(g1["grads"], g2["grads"]):
        assert np.array_equal(a, b)


def test_two_steps_match_oracle():
    # gradient reset after step, dropout step counter advance, and SGD over two steps
    layers = C.resmlp_stack(2, 128, dropout=0.2)
    x, t, params = make_case(layers, 16, 9, "fp32")
    g, P = gpu_step(layers, params, x, t, m=4, n=2, ckpt="except_last", dtype="fp32", lr=0.1, seed=9, steps=2)
    r1 = oracle_step(layers, params, x, t, lr=0.1, m=4, seed=9, step=0)
    r2 = oracle_step(layers, r1["params"], x, t, lr=0.1, m=4, seed=9, step=1)
    errs, bad = compare(g[1], r2, r1["params"], 1e-4, 0.1, gpu_base=g[0]["params"])
    assert not bad, bad


def test_c4_full_width_parity():
    # BASELINE config 4 at full size (U-MLP d = 2048, batch 256, m = 32, 8 partitions with the a1
    # balance [2, 3, ..., 3]: 4 long skip routes, 8-row micro-batches), all partitions on cuda:0 --
    # the multi-GPU code path with same-device copies
    cfg = C.C4()
    gpu, ref, errs, P = _check(cfg.layers, cfg.batch, cfg.m, cfg.n, cfg.checkpoint, cfg.dtype, cfg.lr, cfg.balance)
    from oracle.schedule import SKIP_F, route_partitions, records
    want = records(cfg.m, cfg.n, cfg.checkpoint, route_partitions(cfg.layers, cfg.balance))
    assert np.array_equal(gpu["log"], want)
    assert int((gpu["log"][:, 2] == SKIP_F).sum()) == 4 * cfg.m
