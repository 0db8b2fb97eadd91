"""Table 1 ablation toggles on the GPU: the three design
components torchgpipe adds -- Fork/Join backward order, copy streams, portals -- can each be
switched off.  Switching them off changes only WHEN and HOW the messages move, never the
arithmetic: loss, y, dx, gradients and updated parameters must stay bitwise equal to the default
run, the runtime must issue exactly tgp_schedule_ablation's records, and the relay must move
(d - s) times the portal's skip bytes and hold its extra relay slots in memory."""
import numpy as np
import pytest

from oracle.schedule import route_partitions
from synth import configs as C

from _gpu import gpu_step, make_case

pytestmark = pytest.mark.gpu

LAYERS = C.umlp(d=256)
BAL = [2, 3, 3, 3, 3, 3, 3, 3]
B, M, N = 32, 4, 8


def _run(opts, ckpt="except_last", dtype="bf16"):
    x, t, params = make_case(LAYERS, B, 5, dtype)
    rec, P = gpu_step(LAYERS, params, x, t, m=M, n=N, ckpt=ckpt, dtype=dtype, lr=0.05, balance=BAL, seed=5,
                      options=opts)
    return rec, P


def _same(a, b):
    assert a["loss"] == b["loss"]
    assert np.array_equal(a["y"], b["y"]) and np.array_equal(a["dx"], b["dx"])
    for g, h in zip(a["grads"], b["grads"]):
        assert np.array_equal(g, h)
    for p, q in zip(a["params"], b["params"]):
        assert np.array_equal(p, q)


ROWS = {  # Table 1 rows, top to bottom (the last is the default design)
    "none": {"ablate_order": 11, "ablate_copy_streams": 1, "ablate_portals": 1},
    "dependency": {"ablate_copy_streams": 1, "ablate_portals": 1},
    "dependency+streams": {"ablate_portals": 1},
}


@pytest.mark.parametrize("row", list(ROWS))
def test_ablation_rows_bitwise_equal_to_default(row):
    ref, P0 = _run({})
    got, P = _run(ROWS[row])
    _same(ref, got)
    routes = route_partitions(LAYERS, BAL)
    from paper_2004_09910_b200 import tgp
    want = tgp.schedule(M, N, "except_last", routes, relay=bool(ROWS[row].get("ablate_portals")),
                        order_seed=ROWS[row].get("ablate_order", 0))
    assert np.array_equal(got["log"], want)


@pytest.mark.parametrize("ckpt", ["always", "never"])
def test_unordered_backward_each_mode(ckpt):
    ref, _ = _run({}, ckpt=ckpt)
    got, _ = _run({"ablate_order": 3}, ckpt=ckpt)
    _same(ref, got)


def test_copy_streams_fp32():
    ref, _ = _run({}, dtype="fp32")
    got, _ = _run({"ablate_copy_streams": 1, "ablate_order": 2}, dtype="fp32")
    _same(ref, got)


def test_relay_copy_bytes_and_memory():
    _, Pp = _run({})
    _, Pr = _run({"ablate_portals": 1})
    bp, np_ = Pp.copy_stats()
    br, nr = Pr.copy_stats()
    routes = route_partitions(LAYERS, BAL)
    w = 256  # every route carries the d = 256 residual stream
    per_mb = B // M
    # forward skips in bf16 (2 B), skip gradients fp32 (4 B); per micro-batch and hop
    extra_hops = sum(d - s - 1 for s, d in routes if d > s)
    assert br - bp == extra_hops * M * per_mb * w * (2 + 4)
    assert nr - np_ == extra_hops * M * 2
    # relay slots live on the partitions strictly inside each route
    for j in range(N):
        inside = sum(1 for s, d in routes if s - 1 < j < d - 1)
        dm = Pr.memory(j)["used"] - Pp.memory(j)["used"]
        assert dm == inside * B * w * (2 + 4), (j, dm)
    Pr.set_option("ablate_portals", 0)  # frees them again
    assert all(Pr.memory(j)["used"] == Pp.memory(j)["used"] for j in range(N))
