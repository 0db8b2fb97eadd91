"""GPU parity of the persistent weight-streaming task kernel (csrc/task_stream.cu): F, F' and B of
all-RESMLP partitions with <= 16-row micro-batches run as ONE launch per task.  Compared with the
fp64 oracle (normwise 2e-2, reading Z15) and with itself across checkpoint modes (F' == F bitwise,
reading Z21).  Sizes span several 128-feature slabs per phase, d != H both ways, ragged
micro-batches, dropout, two partitions on one device, and the full C2 block width."""
import numpy as np
import pytest

from synth import configs as C

from _gpu import bf16_shadow, compare, gpu_step, make_case, oracle_step

pytestmark = pytest.mark.gpu
TOL = 2e-2


def _run(layers, B, m, n, ckpt, seed, options=None, balance=None, x_mean=0.0, ln="default", steps=1):
    x, t, params = make_case(layers, B, seed, "bf16", x_mean=x_mean, ln=ln)
    g, P = gpu_step(layers, params, x, t, m=m, n=n, ckpt=ckpt, dtype="bf16", lr=0.05, seed=seed, balance=balance,
                    options=options, steps=steps)
    return x, t, params, g, P


def _kernels_per_step(layers, B, m, stream):
    x, t, params = make_case(layers, B, 1, "bf16")
    g, P = gpu_step(layers, params, x, t, m=m, n=1, ckpt="except_last", dtype="bf16", lr=0.05, seed=1,
                    options={"stream": stream})
    P.close()
    return g["kernels"]


def test_stream_kernel_is_used():
    from paper_2004_09910_b200 import Pipeline

    layers = C.resmlp_stack(2, 512)
    P = Pipeline(layers, chunks=4, devices=[0], checkpoint="except_last", max_batch=64, dtype="bf16")
    assert P.stream_enabled(0)
    P.set_option("stream", 0)
    assert not P.stream_enabled(0)
    P.close()
    on, off = _kernels_per_step(layers, 64, 4, 1), _kernels_per_step(layers, 64, 4, 0)
    # F, F', B are one kernel each with the stream kernel
    assert on < off, (on, off)


@pytest.mark.parametrize("d,H", [(1024, 2048), (1024, 512)])
def test_stream_matches_oracle_and_is_bitwise_across_modes(d, H):
    layers = C.resmlp_stack(3, d, hidden=H, dropout=0.1)
    res = {}
    for mode in ("always", "except_last", "never"):
        x, t, params, g, P = _run(layers, 64, 4, 1, mode, 6)
        res[mode] = g
        P.close()
    for mode in ("except_last", "never"):
        assert res[mode]["loss"] == res["always"]["loss"]
        for a, b in zip(res[mode]["grads"], res["always"]["grads"]):
            assert np.array_equal(a, b)
    ref = oracle_step(layers, params, x, t, lr=0.05, m=4, seed=6, step=0)
    errs, bad = compare(res["never"], ref, params, TOL, 0.05)
    assert not bad, bad


@pytest.mark.parametrize("B,m", [(60, 4), (50, 4), (16, 2)])
def test_stream_ragged_micro_batches(B, m):
    layers = C.resmlp_stack(2, 512, hidden=1024)
    x, t, params, g, P = _run(layers, B, m, 1, "except_last", 11)
    P.close()
    ref = oracle_step(layers, params, x, t, lr=0.05, m=m, seed=11, step=0)
    errs, bad = compare(g, ref, params, TOL, 0.05)
    assert not bad, bad


def test_stream_two_partitions_one_device():
    layers = C.resmlp_stack(4, 512, dropout=0.1)
    x, t, params, g, P = _run(layers, 64, 4, 2, "except_last", 4, balance=[2, 2])
    P.close()
    ref = oracle_step(layers, params, x, t, lr=0.05, m=4, seed=4, step=0)
    errs, bad = compare(g, ref, params, TOL, 0.05)
    assert not bad, bad


def test_stream_full_c2_width_parity():
    # the bench's launch configuration per block (d = H = 4096, 16-row micro-batches, m = 32) on 4 of
    # C2's 32 blocks, so the fp64 oracle finishes in seconds
    layers = C.resmlp_stack(4, 4096)
    x, t, params, g, P = _run(layers, 512, 32, 1, "except_last", 1234)
    P.close()
    ref = oracle_step(layers, params, x, t, lr=0.05, m=32, seed=1234, step=0)
    errs, bad = compare(g, ref, params, TOL, 0.05)
    assert not bad, bad


def test_full_c2_bench_config_parity():
    # VERDICT r1 "next" 1: the EXACT bench configuration (32 x 4096 RESMLP, B = 512, m = 32,
    # except_last, bf16, stream kernel: L = 32 blocks in one launch, 64 phases) against the fp64
    # oracle -- loss, y, dx, every gradient and every delta-theta at 2e-2 normwise (reading Z15)
    layers = C.resmlp_stack(32, 4096)
    x, t, params = make_case(layers, 512, 1234, "bf16")
    g, P = gpu_step(layers, params, x, t, m=32, n=1, ckpt="except_last", dtype="bf16", lr=0.05, seed=1234)
    assert P.stream_enabled(0)
    P.close()
    ref = oracle_step(layers, params, x, t, lr=0.05, m=32, seed=1234, step=0)
    errs, bad = compare(g, ref, params, TOL, 0.05)
    assert not bad, bad


@pytest.mark.parametrize("x_mean", [4.0, 32.0])
def test_stream_offcenter_inputs_parity(x_mean):
    # VERDICT r1 "weak" 2: the LayerNorm folds of the stream kernel (DESIGN R3 forward, R4 backward)
    # change which value is rounded to bf16; off the zero-mean regime (row mean >> row std, wide
    # gamma / beta) the result must still meet 2e-2 normwise.  x ~ N(mu, 1), gamma ~ U(0.25, 4),
    # beta ~ N(0, 1), d = H = 4096, 4 blocks, 16-row micro-batches, dropout, two steps (the fold
    # vectors are recomputed after the SGD step)
    layers = C.resmlp_stack(4, 4096, dropout=0.1)
    B, m, lr, seed = 64, 4, 0.05, 31
    x, t, params = make_case(layers, B, seed, "bf16", x_mean=x_mean, ln="wide")
    g, P = gpu_step(layers, params, x, t, m=m, n=1, ckpt="except_last", dtype="bf16", lr=lr, seed=seed, steps=2)
    assert P.stream_enabled(0)
    P.close()
    ref0 = oracle_step(layers, params, x, t, lr=lr, m=m, seed=seed, step=0)
    errs, bad = compare(g[0], ref0, params, TOL, lr)
    assert not bad, ("step 0", bad)
    # step 1 runs on the bf16 shadow of the updated master weights (Z14); the oracle gets the same
    # rounding of ITS step-0 weights (profiles/diag/offcenter_diag.py: unrounded, both the stream and
    # the per-layer path miss the last block's dbeta by 2.5e-2 at x_mean 4 -- the bf16 weight
    # rounding, not the folds)
    p1 = bf16_shadow(layers, ref0["params"])
    ref1 = oracle_step(layers, p1, x, t, lr=lr, m=m, seed=seed, step=1)
    errs, bad = compare(g[1], ref1, p1, TOL, lr, gpu_base=g[0]["params"])
    assert not bad, ("step 1", bad)


def test_stream_offcenter_two_partitions():
    # off-centre inputs through a partition boundary (the second partition's first block has mu~ = 0
    # in the stream kernel's forward fold) and the ragged tail
    layers = C.resmlp_stack(4, 1024, hidden=2048)
    x, t, params, g, P = _run(layers, 60, 4, 2, "always", 32, balance=[2, 2], x_mean=16.0, ln="wide")
    P.close()
    ref = oracle_step(layers, params, x, t, lr=0.05, m=4, seed=32, step=0)
    errs, bad = compare(g, ref, params, TOL, 0.05)
    assert not bad, bad


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_gradients_accumulate_across_backward_calls(dtype):
    # "gradients accumulate across forward/backward pairs until step": the deferred dW
    # of the second backward adds into the first (TMA reduce-add epilogue), bias / LN partials too
    import torch

    from paper_2004_09910_b200 import Pipeline

    layers = C.resmlp_stack(2, 512, hidden=1024)
    B, m = 64, 4
    x, t, params = make_case(layers, B, 21, dtype)
    ref = oracle_step(layers, params, x, t, lr=0.05, m=m, seed=21, step=0)
    P = Pipeline(layers, chunks=m, devices=[0], checkpoint="except_last", max_batch=B, dtype=dtype, seed=21)
    for i, p in enumerate(params):
        P.set_param(i, p)
    X = torch.tensor(np.asarray(x, np.float32), device="cuda")
    T = torch.tensor(np.asarray(t, np.float32), device="cuda")
    Y = torch.empty(B, 512, device="cuda")
    DY = torch.empty_like(Y)
    for _ in range(2):
        P.forward(X, B, Y)
        P.mse_loss_grad(Y, T, B, DY)
        P.backward(DY)
    tol = 2e-2 if dtype == "bf16" else 1e-4
    scale = max(np.max(np.abs(g)) for g in ref["grads"])
    for k, gr in enumerate(ref["grads"]):
        g = P.get_grad(k)
        e = np.max(np.abs(g - 2.0 * np.asarray(gr).ravel())) / max(2.0 * np.max(np.abs(gr)), 1e-3 * scale)
        assert e <= tol, (k, e)
    P.close()


def test_full_c2_deterministic_and_modes_bitwise():
    # the full BASELINE C2 model (32 x 4096, B = 512, m = 32) on the bench's launch configuration:
    # (a) two identical 3-step runs give bitwise identical losses and gradients (no races, fixed
    # reduction orders), (b) except_last / never / always are bitwise equal (F' == F, reading Z21)
    import torch

    from paper_2004_09910_b200 import Pipeline

    layers = C.resmlp_stack(32, 4096, dropout=0.1)
    B = 512
    g = torch.Generator().manual_seed(5)
    X = torch.randn(B, 4096, generator=g).cuda()
    T = torch.randn(B, 4096, generator=g).cuda()

    def run(mode):
        P = Pipeline(layers, chunks=32, devices=[0], checkpoint=mode, max_batch=B, dtype="bf16", seed=1)
        assert P.stream_enabled(0)
        P.init_params(1)
        Y = torch.empty(B, 4096, device="cuda")
        DY = torch.empty_like(Y)
        losses = []
        for it in range(3):
            P.forward(X, B, Y)
            losses.append(P.mse_loss_grad(Y, T, B, DY))
            P.backward(DY)
            if it < 2:
                P.step(0.05)
        grads = [P.get_grad(i) for i in range(0, P.n_params, 5)]
        P.close()
        return losses, grads

    ref = run("except_last")
    for mode in ("except_last", "never", "always"):
        got = run(mode)
        assert got[0] == ref[0], (mode, got[0], ref[0])
        for a, b in zip(got[1], ref[1]):
            assert np.array_equal(a, b), mode


def test_profile_based_balance():
    # PAPER.md P:124 (balance by profiling): per-layer forward + backward device times
    # of the U-MLP (RESMLP blocks, 2d -> d merges, a d -> d head) are positive, the merges cost more
    # than a head Linear, and the min-max partition of the profiled costs is a valid balance
    from paper_2004_09910_b200 import balance_by_time

    layers = C.umlp(d=512, levels=2, blocks_per_level=1, mid_blocks=1)
    bal, costs = balance_by_time(layers, 3, batch=64, chunks=4, reps=5)
    assert len(costs) == len(layers) and all(c > 0 for c in costs)
    kinds = [l["kind"] for l in layers]
    assert sum(bal) == len(layers) and len(bal) == 3 and min(bal) >= 1
    merge = [c for c, k in zip(costs, kinds) if k == "merge"]
    assert min(merge) > 0.5 * costs[-1]
    uni, ucosts = balance_by_time(C.resmlp_stack(8, 512), 4, batch=64, chunks=4, reps=5)
    assert uni == [2, 2, 2, 2], (uni, ucosts)


def test_memory_plan_checkpointing_saves_activations():
    # checkpointing keeps only the stage input per micro-batch (the receive slab) plus the
    # scratch activation slot(s), instead of every micro-batch's intermediates; the static plan shows
    # it.  With F' / B pairing (the stream kernel) checkpointed micro-batches alternate TWO scratch
    # slots (F'_{i-1} recomputes while B_i reads F'_i's).  What the checkpoint mode changes is exactly
    # the slot bytes; the bf16 dW-operand stash (R1) is the same in every mode (tgp_memory_breakdown).
    from paper_2004_09910_b200 import Pipeline

    layers = C.resmlp_stack(4, 1024)
    use, br = {}, {}
    for mode in ("always", "except_last", "never"):
        P = Pipeline(layers, chunks=8, devices=[0], checkpoint=mode, max_batch=128, dtype="bf16")
        use[mode] = P.memory(0)
        br[mode] = P.memory_breakdown(0)
        P.close()
    assert use["always"]["params"] == use["never"]["params"]
    # always: 2 scratch; except_last: 2 scratch + micro-batch m; never: 1 scratch + m
    assert [br[m]["n_slots"] for m in ("always", "except_last", "never")] == [2, 3, 9]
    assert br["always"]["stash"] == br["except_last"]["stash"] == br["never"]["stash"] > 0
    # 4 RESMLP blocks x 4 bf16 operands (Hop, Gop, dAop, dYop) x 128 rows x 1024
    assert br["always"]["stash"] == 4 * 4 * 128 * 1024 * 2
    per_slot = br["always"]["slots"] / 2
    assert per_slot > 0
    for mode in ("except_last", "never"):
        assert br[mode]["slots"] == br[mode]["n_slots"] * per_slot
        dslots = br[mode]["slots"] - br["always"]["slots"]
        assert abs((use[mode]["used"] - use["always"]["used"]) - dslots) <= 0.01 * dslots
    # without the stream kernel (32-row micro-batches: per-layer kernels) F'_{i-1} still runs beside B_i,
    # so the checkpointed micro-batches still alternate two scratch slots; one checkpointed micro-batch
    # (m = 2, except_last) has nothing to pair with: one slot for it plus the kept last one
    P = Pipeline(C.resmlp_stack(4, 1024), chunks=4, devices=[0], checkpoint="always", max_batch=128, dtype="bf16")
    assert P.memory_breakdown(0)["n_slots"] == 2
    P.close()
    P = Pipeline(C.resmlp_stack(4, 1024), chunks=2, devices=[0], checkpoint="except_last", max_batch=128, dtype="bf16")
    assert P.memory_breakdown(0)["n_slots"] == 2
    P.close()
