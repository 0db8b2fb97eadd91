"""GPU tests of F' / B pairing (option "pair_recompute", runtime.cu issue()): the recompute F'_{i-1,j}
depends only on the stage input and the weights, not on B_{i,j}, so it runs on
a second compute lane beside B_{i,j}: persistent task kernels on half grids (each cluster owns two
output slabs), or -- on partitions that run the per-layer kernels -- full-size kernels sharing the SMs.

* Results are BITWISE equal with and without pairing (a half-grid task computes every output with the
  same split-K order and fixed-order reductions as the full grid; reading Z21), over checkpoint
  modes, d != H both ways (half-grid units without work), dropout, ragged micro-batches, several
  partitions on one device, and the full C2 block width.
* The device timeline keeps the dependencies: B tasks in the paper's order on lane 0, every F'_i ends
  before B_i starts, a hoisted F'_{i-1} starts only after B_{i+1} ended (its scratch slot's last
  reader), and F' really overlaps B."""
import numpy as np
import pytest

from synth import configs as C

from _gpu import gpu_step, make_case

pytestmark = pytest.mark.gpu


def _both(layers, B, m, n, ckpt, seed=4, steps=2, option="pair_recompute"):
    x, t, params = make_case(layers, B, seed, "bf16")
    res = {}
    for pair in (0, 1):
        g, P = gpu_step(layers, params, x, t, m=m, n=n, ckpt=ckpt, dtype="bf16", lr=0.05, seed=seed,
                        options={option: pair}, steps=steps)
        res[pair] = g if steps > 1 else [g]
        P.close()
    for a, b in zip(res[0], res[1]):
        assert a["loss"] == b["loss"]
        assert np.array_equal(a["y"], b["y"])
        assert np.array_equal(a["dx"], b["dx"])
        for k, (ga, gb) in enumerate(zip(a["grads"], b["grads"])):
            assert np.array_equal(ga, gb), k
        for k, (pa, pb) in enumerate(zip(a["params"], b["params"])):
            assert np.array_equal(pa, pb), k
        assert a["log"].tolist() == b["log"].tolist()  # the issue log keeps the paper's schedule


@pytest.mark.parametrize("ckpt", ["except_last", "always"])
def test_pairing_bitwise_two_partitions(ckpt):
    _both(C.resmlp_stack(4, 512, hidden=1024, dropout=0.1), 64, 4, 2, ckpt)


@pytest.mark.parametrize("d,H", [(1024, 2048), (1024, 512)])
def test_pairing_bitwise_d_ne_h_ragged(d, H):
    # 60 rows in 5 micro-batches of 12; d != H: on the half grid some (phase, slab) units are empty
    _both(C.resmlp_stack(3, d, hidden=H, dropout=0.1), 60, 5, 1, "except_last")


def test_pairing_bitwise_full_c2_width():
    _both(C.resmlp_stack(4, 4096), 512, 32, 1, "except_last", steps=1)


@pytest.mark.parametrize("ckpt", ["except_last", "always"])
def test_pairing_bitwise_per_layer_kernels(ckpt):
    # 64-row micro-batches: the per-layer tcgen05 GEMMs (no stream kernel); F'_{i-1} runs on lane 1
    # with full-size kernels beside B_i, two partitions on one device
    _both(C.resmlp_stack(4, 512, hidden=1024, dropout=0.1), 256, 4, 2, ckpt)


def test_pairing_bitwise_per_layer_portals():
    # a U-MLP with skip routes (MERGE layers pop the portal tensors in F and F'); the GPT-2-shaped stack
    # is covered by test_gpu_gpt2.py::test_c5_checkpoint_modes_bitwise (paired always / except_last == never)
    _both(C.umlp(d=256, levels=2, blocks_per_level=1, mid_blocks=1), 64, 2, 2, "always")


@pytest.mark.parametrize("rows", [64, 256])
def test_checkpointed_f_without_dead_stores_is_bitwise(rows):
    # option "dead_stash": a checkpointed F stores only its output (F' recomputes the intermediates):
    # bitwise equal to storing everything, on the stream kernel (16-row micro-batches) and the
    # per-layer kernels (64-row micro-batches)
    _both(C.resmlp_stack(4, 512, hidden=1024, dropout=0.1), rows, 4, 2, "always", option="dead_stash")


def test_pairing_dependencies_on_the_device_timeline():
    import torch

    from oracle.schedule import B as KB, RECOMPUTE

    layers = C.resmlp_stack(4, 1024)
    m, n, Bt = 8, 2, 128
    x, t, params = make_case(layers, Bt, 2, "bf16")
    g, P = gpu_step(layers, params, x, t, m=m, n=n, ckpt="except_last", dtype="bf16", lr=0.05, steps=1)
    P.set_trace(True)
    X = torch.tensor(x, device="cuda")
    T = torch.tensor(t, device="cuda")
    Y = torch.empty(Bt, 1024, device="cuda")
    DY = torch.empty_like(Y)
    P.forward(X, Bt, Y)
    P.mse_loss_grad(Y, T, Bt, DY)
    P.backward(DY)
    tl = P.timeline()
    P.close()
    overlaps = 0
    for j in range(n):
        rows = tl[tl[:, 0] == j]
        b = {int(r[3]): (int(r[4]), int(r[5])) for r in rows if int(r[2]) == KB and int(r[1]) == 0}
        f = {int(r[3]): (int(r[4]), int(r[5])) for r in rows if int(r[2]) == RECOMPUTE}
        lanes = {int(r[3]): int(r[1]) for r in rows if int(r[2]) == RECOMPUTE}
        assert sorted(b) == list(range(1, m + 1)) and sorted(f) == list(range(1, m))
        assert all(lanes[i] == 3 for i in f)  # every F' ran on lane 1
        starts = [b[i][0] for i in range(m, 0, -1)]
        assert starts == sorted(starts)  # B_m, ..., B_1 in order
        slack = 2000  # ns of event resolution
        for i in f:
            assert f[i][1] <= b[i][0] + slack, (j, i)             # F'_i before B_i
            if i + 2 <= m:
                assert f[i][0] + slack >= b[i + 2][1], (j, i)     # after B_{i+2} (same scratch slot)
            if i + 1 <= m and f[i][0] < b[i + 1][1] and b[i + 1][0] < f[i][1]:
                overlaps += 1                                      # F'_i beside B_{i+1}
    assert overlaps >= n * (m - 2)
