"""GPU tests of compute fused with send (option "fused_send"; PAPER.md P:137 two-way
synchronisation, P:198-203 copy streams): a persistent stream-kernel task stores its boundary tensor
-- F_{i,j}: the last block's output, B_{i,j}: the input gradient -- straight into the neighbouring
partition's receive slab and release-stores the receive flag itself (system scope), so the
COPY_F / COPY_B records launch no copy kernel.

* Results are BITWISE equal to the push-kernel transport (the same bytes land in the same slab),
  with pairing, dropout, several partitions per device and the full C2 block width.
* The copy kernels disappear: 2 m (n - 1) fewer kernels per step; the copied bytes are unchanged.
* The receive waits still guard the data: with every receive slab poisoned with NaN before each
  forward call, the fused path gives the same bits."""
import numpy as np
import pytest

from synth import configs as C

from _gpu import gpu_step, make_case

pytestmark = pytest.mark.gpu


def _run(layers, B, m, n, ckpt, options, steps=2, seed=6):
    x, t, params = make_case(layers, B, seed, "bf16")
    g, P = gpu_step(layers, params, x, t, m=m, n=n, ckpt=ckpt, dtype="bf16", lr=0.05, seed=seed, options=options,
                    steps=steps)
    stats = P.copy_stats()
    P.close()
    return (g if steps > 1 else [g]), stats


def _same(a, b):
    for ra, rb in zip(a, b):
        assert ra["loss"] == rb["loss"]
        assert np.array_equal(ra["y"], rb["y"]) and np.array_equal(ra["dx"], rb["dx"])
        for k, (ga, gb) in enumerate(zip(ra["grads"], rb["grads"])):
            assert np.array_equal(ga, gb), k
        for k, (pa, pb) in enumerate(zip(ra["params"], rb["params"])):
            assert np.array_equal(pa, pb), k
        assert ra["log"].tolist() == rb["log"].tolist()


@pytest.mark.parametrize("ckpt,n", [("except_last", 2), ("always", 4)])
def test_fused_send_bitwise_and_no_copy_kernels(ckpt, n):
    layers = C.resmlp_stack(8, 512, hidden=1024, dropout=0.1)
    m, B = 8, 128
    push, s_push = _run(layers, B, m, n, ckpt, {"fused_send": 0, "transport": 0})
    fused, s_fused = _run(layers, B, m, n, ckpt, {"fused_send": 1})
    _same(push, fused)
    assert s_push == s_fused  # same messages and bytes
    # kernels of the second step: the push kernels are gone
    assert push[1]["kernels"] - push[0]["kernels"] - (fused[1]["kernels"] - fused[0]["kernels"]) == 2 * m * (n - 1)


def test_fused_send_full_c2_width():
    layers = C.resmlp_stack(4, 4096)
    push, _ = _run(layers, 512, 32, 2, "except_last", {"fused_send": 0, "transport": 0}, steps=1)
    fused, _ = _run(layers, 512, 32, 2, "except_last", {"fused_send": 1}, steps=1)
    _same(push, fused)


def test_fused_send_receive_waits_still_guard_the_slab():
    layers = C.resmlp_stack(4, 512)
    ref, _ = _run(layers, 64, 4, 4, "except_last", {"fused_send": 0, "transport": 0})
    poisoned, _ = _run(layers, 64, 4, 4, "except_last", {"fused_send": 1, "test_poison": 1})
    _same(ref, poisoned)
    assert all(np.isfinite(r["y"]).all() for r in poisoned)
