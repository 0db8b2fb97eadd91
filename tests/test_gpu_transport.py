"""Boundary robustness and the stage-boundary transports (VERDICT r1 "next" 4 and 5).

* Watchdog ("a handshake wait past the watchdog -> TGP_E_TIMEOUT", the
  host issues and the device waits): a lost forward message makes the consumer's stream wait forever
  in cuStreamWaitValue32; the call must return TGP_E_TIMEOUT (-6) after `watchdog_ms` instead of
  hanging (the release of the waits is attempted; on B200 a pending stream-memory wait can keep the
  release kernel from running, so the child process exits instead of reusing the device) and fail
  the context (TGP_E_STATE afterwards).
* Copy-engine transport (option "transport" = 1: cudaMemcpyAsync + cuStreamWriteValue32, PAPER.md
  P:198-203 copy streams) moves the same bytes as the SM push kernel: results bitwise equal.
* tgp_bench_transport: per-message device time of both transports."""
import time

import numpy as np
import pytest

from synth import configs as C

from _gpu import compare, gpu_step, make_case, oracle_step

pytestmark = pytest.mark.gpu


def _pipe(layers, n, B, m, **kw):
    from paper_2004_09910_b200 import Pipeline

    return Pipeline(layers, chunks=m, devices=[0] * n, balance=kw.get("balance"), checkpoint="except_last",
                    max_batch=B, dtype=kw.get("dtype", "bf16"), seed=3)


_WD_CHILD = r"""
import json, os, sys, time
sys.path.insert(0, sys.argv[1])
import torch
from paper_2004_09910_b200 import Pipeline, TgpError
from synth import configs as C
layers = C.resmlp_stack(4, 256, hidden=512)
B, m = 32, 4
P = Pipeline(layers, chunks=m, devices=[0, 0], balance=[2, 2], checkpoint="except_last", max_batch=B,
             dtype="bf16", seed=3)
P.init_params(3)
P.set_option("watchdog_ms", 1500)
P.set_option("test_drop_push", 0)  # partition 0 never sends x_i^1: partition 1 would wait forever
X = torch.randn(B, 256, device="cuda")
Y = torch.empty(B, 256, device="cuda")
out = {}
t0 = time.time()
try:
    P.forward(X, B, Y)
    out["rc"] = 0
except TgpError as e:
    out["rc"], out["msg"] = e.rc, str(e)
out["elapsed"] = time.time() - t0
try:
    P.forward(X, B, Y)
    out["rc2"] = 0
except TgpError as e:
    out["rc2"] = e.rc
P.close()  # a wedged device: destroy must not block either
out["closed"] = True
print(json.dumps(out), flush=True)
os._exit(0)  # process exit reclaims whatever the device still holds
"""


def test_watchdog_returns_timeout_on_lost_message():
    # in a child process: a wedged device must not take the test session with it
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _WD_CHILD, root], capture_output=True, text=True, timeout=240)
    line = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert line, (r.returncode, r.stdout[-2000:], r.stderr[-2000:])
    out = json.loads(line[-1])
    assert out["rc"] == -6 and "watchdog" in out["msg"], out
    assert out["elapsed"] < 30, out
    assert out["rc2"] == -2 and out["closed"], out


def test_watchdog_does_not_fire_on_slow_healthy_calls():
    # a delayed (not lost) message completes inside the bound: no false positive
    import torch

    layers = C.resmlp_stack(4, 256, hidden=512)
    B, m = 32, 4
    P = _pipe(layers, 2, B, m, balance=[2, 2])
    P.init_params(3)
    P.set_option("watchdog_ms", 5000)
    P.set_option("test_delay_push_us", 200)
    X = torch.randn(B, 256, device="cuda")
    Y = torch.empty(B, 256, device="cuda")
    P.forward(X, B, Y)
    P.close()


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_copy_engine_transport_bitwise_and_parity(dtype):
    # 4 partitions with skip routes (C4-shaped U-MLP): COPY_F / COPY_B through the copy engine, skips
    # through the push kernel; every result bitwise equal to the SM push transport, and oracle parity
    layers = C.umlp(d=256, levels=2, blocks_per_level=1, mid_blocks=1)
    B, m, n = 32, 4, 4
    x, t, params = make_case(layers, B, 12, dtype)
    res = {}
    for tr in (0, 1, 2):
        g, P = gpu_step(layers, params, x, t, m=m, n=n, ckpt="except_last", dtype=dtype, lr=0.05, seed=12,
                        options={"transport": tr})
        res[tr] = g
        P.close()
    for tr in (1, 2):
        assert res[0]["loss"] == res[tr]["loss"]
        assert np.array_equal(res[0]["y"], res[tr]["y"]) and np.array_equal(res[0]["dx"], res[tr]["dx"])
        for a, b in zip(res[0]["grads"], res[tr]["grads"]):
            assert np.array_equal(a, b)
    ref = oracle_step(layers, params, x, t, lr=0.05, m=m, seed=12, step=0)
    errs, bad = compare(res[1], ref, params, 2e-2 if dtype == "bf16" else 1e-4, 0.05)
    assert not bad, bad


def test_bench_transport_both_modes():
    from paper_2004_09910_b200 import bench_transport

    for nbytes in (4096, 262144, 4 << 20):
        for mode in (0, 1):
            us, pp = bench_transport(0, 0, nbytes, mode, reps=20)
            assert 0.0 < us < 1e4 and 0.0 < pp < 1e4, (nbytes, mode, us, pp)
