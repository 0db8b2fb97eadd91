"""Multi-process pipeline (one process per partition, torchrun, CUDA-IPC receive arenas) vs the
oracle.  On a 1-GPU box all ranks share cuda:0; the transport code path is the multi-GPU one."""
import os
import subprocess
import sys

import numpy as np
import pytest

from synth import configs as C
from synth import gen as G

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(world, cfg, tmp_path):
    port = 29500 + (os.getpid() % 1000)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "tests", "mp_worker.py"),
           str(tmp_path), cfg]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=240)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return [dict(np.load(os.path.join(tmp_path, f"rank{k}.npz"))) for k in range(world)]


@pytest.mark.parametrize("world,cfg", [(2, "resmlp"), (4, "resmlp"), (3, "umlp"), (2, "stream"), (3, "gpt2")])
def test_multiprocess_matches_oracle(world, cfg, tmp_path):
    from oracle import model as OM
    res = _run(world, cfg, tmp_path)
    if cfg == "umlp":
        layers = C.umlp(d=256, levels=2, blocks_per_level=1, mid_blocks=1)
    elif cfg == "gpt2":
        layers = C.gpt2_stack(3, 128, 2, 64, 512, 0.1)
    else:
        layers = C.resmlp_stack(2 * world, 512 if cfg == "stream" else 256, dropout=0.1)
    B, m, lr, seed = (64 if cfg == "stream" else 32), 4, 0.05, 11
    x, t = G.inputs(layers, 4 if cfg == "gpt2" else B, seed=seed, dtype="bf16")
    if cfg == "gpt2":
        m = 2
    params = G.params(layers, seed=seed, dtype="bf16")
    ref = OM.train_step(layers, params, x, t, lr=lr, m=m, seed=seed, step=0)
    last = res[-1]
    assert abs(float(last["loss0"]) - ref["loss"]) <= 2e-2 * ref["loss"]
    assert np.max(np.abs(last["y0"] - ref["y"])) <= 2e-2 * np.max(np.abs(ref["y"]))
    if cfg != "gpt2":  # (the embedding has no input gradient)
        assert np.max(np.abs(res[0]["dx0"] - ref["dx"])) <= 2e-2 * np.max(np.abs(ref["dx"]))
    scale = max(np.max(np.abs(g)) for g in ref["grads"])
    seen = set()
    for r in res:
        for k, v in r.items():
            if k.startswith("g0_"):
                i = int(k[3:])
                seen.add(i)
                gr = ref["grads"][i].ravel()
                assert np.max(np.abs(v - gr)) <= 2e-2 * max(np.max(np.abs(gr)), 1e-3 * scale), i
    assert seen == set(range(len(ref["grads"])))
    # the second step ran too (flags / sequence numbers across calls)
    assert np.isfinite(float(last["loss1"])) and float(last["loss1"]) != float(last["loss0"])


def test_multiprocess_c2_n8_matches_oracle(tmp_path):
    # VERDICT r1 "next" 4: the n = 8 per-rank C2 shape -- 8 processes (torchrun), 4 x RESMLP(4096) each,
    # B = 512, m = 32, except_last, stream kernel with F'/B pairing and fused sends through CUDA-IPC
    # receive arenas -- against the fp64 oracle of the whole 32-block model: loss, y, dx at 2e-2
    # normwise, every gradient on a fixed subsample (every 97th element), and a second step
    from oracle import model as OM

    world = 8
    port = 29500 + (os.getpid() % 1000) + 7
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "tests", "mp_worker.py"),
           str(tmp_path), "c2n8"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = [dict(np.load(os.path.join(tmp_path, f"rank{k}.npz"))) for k in range(world)]
    layers = C.resmlp_stack(32, 4096)
    B, m, lr, seed = 512, 32, 0.05, 11
    x, t = G.inputs(layers, B, seed=seed, dtype="bf16")
    params = G.params(layers, seed=seed, dtype="bf16")
    ref = OM.train_step(layers, params, x, t, lr=lr, m=m, seed=seed, step=0)
    last = res[-1]
    assert abs(float(last["loss0"]) - ref["loss"]) <= 2e-2 * ref["loss"]
    assert np.max(np.abs(last["y0"] - ref["y"])) <= 2e-2 * np.max(np.abs(ref["y"]))
    assert np.max(np.abs(res[0]["dx0"] - ref["dx"])) <= 2e-2 * np.max(np.abs(ref["dx"]))
    scale = max(np.max(np.abs(g)) for g in ref["grads"])
    seen = set()
    for rr in res:
        for k, v in rr.items():
            if k.startswith("g0_"):
                i = int(k[3:])
                seen.add(i)
                gr = ref["grads"][i].ravel()[::97]
                assert np.max(np.abs(v - gr)) <= 2e-2 * max(np.max(np.abs(gr)), 1e-3 * scale), i
    assert seen == set(range(len(ref["grads"])))
    assert np.isfinite(float(last["loss1"])) and float(last["loss1"]) != float(last["loss0"])
