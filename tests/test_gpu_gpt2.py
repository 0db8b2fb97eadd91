"""GPU parity of the GPT-2-shaped stack (C5, BASELINE.json configs[4]; SURVEY 8(c) "pinned on shrunk
C5"): embedding, pre-LN causal-attention blocks with dropout, LM head and token cross-entropy,
pipelined through the C ABI, against the fp64 oracle on the same seeded tokens and parameters.
Bar: normwise 2e-2 (bf16, reading Z15) on loss, logits, every gradient and every delta-theta;
checkpoint modes bitwise equal (recompute under the restored Philox counters, reading Z17/Z21)."""
import numpy as np
import pytest

from synth import configs as C

from _gpu import compare, make_case, oracle_step

pytestmark = pytest.mark.gpu


def gpt_step(layers, params, x, t, *, m, n, ckpt, lr, balance=None, seed=0, options=None):
    import torch

    from paper_2004_09910_b200 import Pipeline

    B = x.shape[0]
    P = Pipeline(layers, chunks=m, devices=[0] * n, balance=balance, checkpoint=ckpt, max_batch=B, dtype="bf16",
                 seed=seed)
    for k, v in (options or {}).items():
        P.set_option(k, v)
    for idx, p in enumerate(params):
        P.set_param(idx, p)
    dev = torch.device("cuda", 0)
    X = torch.tensor(np.asarray(x, np.float32), device=dev)
    T = torch.tensor(np.asarray(t, np.int32), device=dev)
    V = layers[-1]["d_out"]
    Y = torch.empty(B, V, device=dev)
    DY = torch.empty(B, V, device=dev)
    DX = torch.zeros(B, 1, device=dev)
    P.forward(X, B, Y)
    loss = P.ce_loss_grad(Y, T, B, DY)
    P.backward(DY, DX)
    rec = dict(loss=loss, y=Y.cpu().numpy().astype(np.float64), dx=np.zeros((B, 1)),
               grads=[P.get_grad(i) for i in range(P.n_params)], log=P.issue_log(), kernels=P.kernel_count())
    P.step(lr)
    rec["params"] = [P.get_param(i) for i in range(P.n_params)]
    if options and "attn_tc" in options:
        P.set_option("attn_tc", -1)  # the switch is process-wide: back to the default
    P.close()
    return rec


def _run(layers, nseq, m, n, ckpt, balance=None, seed=11, lr=0.01, options=None):
    x, t, params = make_case(layers, nseq, seed, "bf16")
    ref = oracle_step(layers, params, x, t, lr=lr, m=m, seed=seed, step=0)
    gpu = gpt_step(layers, params, x, t, m=m, n=n, ckpt=ckpt, lr=lr, balance=balance, seed=seed, options=options)
    errs, bad = compare(gpu, ref, params, 2e-2, lr)
    assert not bad, f"errors above 2e-2: {bad}"
    return gpu, ref, errs


def test_c5_small_parity_always():
    cfg = C.C5_small()  # 4 blocks, d 128, 2 heads, seq 64, V 512, 8 seqs, m 4, n 2, dropout 0.1
    gpu, ref, errs = _run(cfg.layers, cfg.batch, cfg.m, cfg.n, cfg.checkpoint, balance=[3, 3])
    from oracle.schedule import records
    assert np.array_equal(gpu["log"], records(cfg.m, cfg.n, cfg.checkpoint))


def test_c5_no_dropout_single_partition():
    layers = C.gpt2_stack(2, 128, 2, 64, 256, 0.0)
    _run(layers, 2, 1, 1, "never")


def test_c5_wider_multi_tile():
    # d 256 (4 heads), seq 192 (3 attention tiles per sequence), MLP 1024, V 1024, 5 sequences split
    # unevenly over m = 3 micro-batches ([2, 2, 1] sequences), n = 3
    layers = C.gpt2_stack(3, 256, 4, 192, 1024, 0.1)
    _run(layers, 5, 3, 3, "except_last", balance=[2, 1, 2])


def test_c5_checkpoint_modes_bitwise():
    layers = C.gpt2_stack(2, 128, 2, 128, 512, 0.1)
    x, t, params = make_case(layers, 4, 3, "bf16")
    outs = [gpt_step(layers, params, x, t, m=4, n=2, ckpt=mode, lr=0.01, balance=[2, 2], seed=3)
            for mode in ("always", "except_last", "never")]
    for o in outs[1:]:
        assert o["loss"] == outs[0]["loss"]
        assert np.array_equal(o["y"], outs[0]["y"])
        for a, b in zip(o["grads"], outs[0]["grads"]):
            assert np.array_equal(a, b)


def test_c5_ragged_width():
    # d = 320 (5 heads): 3d = 960 and d are not multiples of the 128-row tensor-core tile (full C5's
    # d = 1600 is not either) and the LayerNorm takes the non-cluster path
    layers = C.gpt2_stack(2, 320, 5, 64, 640, 0.1)
    _run(layers, 3, 3, 2, "always", balance=[2, 2])


def test_c5_persistent_wide_gemm_matches_tile_gemm():
    # micro-batches of 2 x 256 tokens: every per-micro-batch GEMM has N = 512 rows and takes the
    # persistent gemm_wide kernel; compare with the one-tile-per-CTA gemm_tc (options off, no
    # split-K) and with the oracle.  (Not bitwise: measured ~1e-6 relative differences between the
    # two kernels' paths; both are deterministic run to run.)
    layers = C.gpt2_stack(2, 256, 4, 256, 512, 0.1)
    x, t, params = make_case(layers, 4, 5, "bf16")
    a = gpt_step(layers, params, x, t, m=2, n=2, ckpt="except_last", lr=0.01, balance=[2, 2], seed=5)
    a2 = gpt_step(layers, params, x, t, m=2, n=2, ckpt="except_last", lr=0.01, balance=[2, 2], seed=5)
    b = gpt_step(layers, params, x, t, m=2, n=2, ckpt="except_last", lr=0.01, balance=[2, 2], seed=5,
                 options={"gemm_wide": 0, "splitk": 1})
    assert a["loss"] == a2["loss"] and all(np.array_equal(u, v) for u, v in zip(a["grads"], a2["grads"]))
    assert abs(a["loss"] - b["loss"]) <= 1e-5 * abs(b["loss"])
    for ga, gb in zip(a["grads"], b["grads"]):
        assert np.max(np.abs(ga - gb)) <= 1e-3 * max(np.max(np.abs(gb)), 1e-12)
    ref = oracle_step(layers, params, x, t, lr=0.01, m=2, seed=5, step=0)
    errs, bad = compare(a, ref, params, 2e-2, 0.01)
    assert not bad, bad


def test_c5_full_width_parity():
    # the full C5 layer shapes (d 1600 = 25 heads x 64, MLP 6400, seq 1024, V 50304; ragged 128-row
    # tiles, 16 attention tiles per sequence, 1024-row micro-batches on the persistent GEMM) on a
    # shortened stack: embed + 2 blocks + LM head, 2 sequences, m = 2, n = 2, dropout 0.1, always
    layers = C.gpt2_stack(2, 1600, 25, 1024, 50304, 0.1)
    _run(layers, 2, 2, 2, "always", balance=[2, 2], seed=21)


def test_c5_split_rows_attention():
    # seq 640 = 10 key tiles: query tiles 8 and 9 are split into two key ranges (partials merged in
    # fixed order); also checked against the checkpoint-free run bitwise (F' == F)
    layers = C.gpt2_stack(2, 128, 2, 640, 512, 0.1)
    gpu, ref, errs = _run(layers, 2, 2, 2, "always", balance=[2, 2], seed=9, options={"attn_tc": 0})
    x, t, params = make_case(layers, 2, 9, "bf16")
    b = gpt_step(layers, params, x, t, m=2, n=2, ckpt="never", lr=0.01, balance=[2, 2], seed=9,
                 options={"attn_tc": 0})
    assert b["loss"] == gpu["loss"] and np.array_equal(b["y"], gpu["y"])


@pytest.mark.parametrize("seq,nh", [(256, 2), (512, 3)])
def test_c5_attention_tcgen05_vs_mma_sync(seq, nh):
    # the tcgen05 attention (default: forward and the dK/dV + dQ backward on 128 x 128 tiles, S, dP
    # and every transposed product on the tensor cores) and the mma.sync kernels (option attn_tc = 0)
    # both against the oracle, and against each other (same arithmetic up to accumulation order)
    layers = C.gpt2_stack(2, 64 * nh, nh, seq, 512, 0.1)
    x, t, params = make_case(layers, 2, 4, "bf16")
    res = {}
    try:
        for tc in (0, 1):
            res[tc] = gpt_step(layers, params, x, t, m=2, n=2, ckpt="always", lr=0.01, balance=[2, 2], seed=4,
                               options={"attn_tc": tc})
    finally:
        from paper_2004_09910_b200 import Pipeline  # reset the process-wide switch
        P = Pipeline(layers, chunks=2, devices=[0, 0], balance=[2, 2], max_batch=x.shape[0], dtype="bf16")
        P.set_option("attn_tc", -1)
        P.close()
    ref = oracle_step(layers, params, x, t, lr=0.01, m=2, seed=4, step=0)
    for tc in (0, 1):
        errs, bad = compare(res[tc], ref, params, 2e-2, 0.01)
        assert not bad, (tc, bad)
    assert abs(res[0]["loss"] - res[1]["loss"]) <= 1e-4 * abs(res[0]["loss"])
    for ga, gb in zip(res[0]["grads"], res[1]["grads"]):
        assert np.max(np.abs(ga - gb)) <= 1e-2 * max(np.max(np.abs(ga)), 1e-12)
