"""CPU (no GPU) tests of the C-ABI library: it loads, exports every symbol include/tgp.h declares,
and its pure host entry points (schedule emitter, balancer, split) agree bit-exactly with the
oracle.  Argument validation of tgp_create happens before any CUDA call."""
import ctypes
import itertools
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2004_09910_b200 import tgp
    if not os.path.exists(tgp.LIB_PATH):
        from paper_2004_09910_b200.build import build
        build(verbose=False)
    return tgp


def test_library_exports_every_header_symbol(L):
    hdr = open(os.path.join(ROOT, "include", "tgp.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    declared = sorted(set(re.findall(r"\b(tgp_[a-z0-9_]+)\s*\(", hdr)))
    assert len(declared) >= 25
    lib = ctypes.CDLL(L.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    # the binding wraps exactly the declared functions
    assert sorted(L.exported_symbols()) == declared


def test_schedule_matches_oracle(L):
    from oracle import schedule as S
    for m, n, mode in itertools.product([1, 2, 3, 4, 8, 32], [1, 2, 3, 4, 8], S.MODES):
        assert np.array_equal(L.schedule(m, n, mode), S.records(m, n, mode)), (m, n, mode)
    for routes in ([(1, 7), (2, 6), (3, 5), (3, 4)], [(1, 4), (1, 4), (2, 2)], [(3, 3)]):
        for m, mode in itertools.product([1, 4, 32], S.MODES):
            got = L.schedule(m, 8, mode, routes)
            assert np.array_equal(got, S.records(m, 8, mode, routes))


def test_balance_matches_oracle(L):
    from oracle import balance as B
    rs = np.random.default_rng(11)
    for trial in range(500):
        Ln = int(rs.integers(1, 40))
        n = int(rs.integers(1, min(8, Ln) + 1))
        costs = [int(v) for v in rs.integers(0, 9, Ln)] if trial % 2 else [float(v) for v in rs.random(Ln)]
        assert L.balance(costs, n) == B.balance_dp(costs, n)


def test_split_matches_oracle(L):
    from oracle import schedule as S
    for B, m in [(8, 4), (10, 4), (512, 32), (7, 7), (100, 3), (1, 1)]:
        assert L.split(B, m) == S.split_sizes(B, m)
    with pytest.raises(L.TgpError):
        L.split(3, 4)


def test_create_validates_before_touching_cuda(L):
    from synth import configs as C
    bad = [
        dict(chunks=0),                     # m < 1
        dict(chunks=20, max_batch=16),      # m > B
        dict(balance=[3, 2]),               # sum(balance) != n_layers
        dict(balance=[4, 0]),               # empty partition
    ]
    for kw in bad:
        args = dict(chunks=4, devices=[0, 0], balance=[2, 2], max_batch=16, dtype="fp32")
        args.update(kw)
        with pytest.raises(L.TgpError) as ei:
            L.Pipeline(C.mlp_chain(4, 64), **args)
        assert "(-1)" in str(ei.value)
    # shape mismatch between consecutive layers
    layers = C.mlp_chain(4, 64)
    layers[2]["d_in"] = 32
    with pytest.raises(L.TgpError):
        L.Pipeline(layers, chunks=2, devices=[0], balance=[4], max_batch=4, dtype="fp32")
    # pop before stash
    layers = C.umlp(d=128, levels=1, blocks_per_level=1, mid_blocks=1)
    layers[0]["stash"], layers[2]["pop"] = -1, 0
    with pytest.raises(L.TgpError):
        L.Pipeline(layers, chunks=2, devices=[0], balance=[len(layers)], max_batch=4, dtype="bf16")
    # fp32 widths must be multiples of 4 (float4 row kernels): rejected at create, with a message
    for d_in, d_out in ((3, 4), (4, 6)):
        layers = [C.layer("linear", d_in, d_out)]
        with pytest.raises(L.TgpError) as ei:
            L.Pipeline(layers, chunks=1, devices=[0], balance=[1], max_batch=4, dtype="fp32")
        assert "(-5)" in str(ei.value) and "multiples of 4" in str(ei.value)


def test_create_validates_gpt2_layers(L):
    # GPT-2-shaped kinds (C5): validation happens before any CUDA call, so it is testable here
    from synth import configs as C

    def make(layers, **kw):
        args = dict(chunks=2, devices=[0], balance=[len(layers)], max_batch=2 * 64, dtype="bf16")
        args.update(kw)
        return L.Pipeline(layers, **args)

    ok = C.gpt2_stack(2, 128, 2, 64, 512, 0.1)
    cases = []
    bad = [dict(L) for L in ok]
    bad[1]["n_heads"] = 3                           # d != 64 * n_heads
    cases.append((bad, {}, "(-1)"))
    bad = [dict(L) for L in ok]
    bad[1]["seq"] = bad[2]["seq"] = 96              # seq % 64 != 0
    cases.append((bad, {}, "(-1)"))
    bad = [dict(L) for L in ok]
    bad[0], bad[1] = bad[1], bad[0]                 # embedding not at layer 0
    cases.append((bad, {}, "(-1)"))
    cases.append((ok, dict(max_batch=100), "(-1)"))  # max_batch not whole sequences
    cases.append((ok, dict(chunks=3), "(-1)"))       # more micro-batches than sequences
    cases.append((ok, dict(dtype="fp32"), "(-5)"))   # bf16 only
    for layers, kw, code in cases:
        with pytest.raises(L.TgpError) as ei:
            make(layers, **kw)
        assert code in str(ei.value), (kw, str(ei.value))


def test_no_cpu_fallback(L):
    # a valid pipeline on a machine without a GPU must fail loudly (TGP_E_CUDA), never fall back
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from synth import configs as C
    with pytest.raises(L.TgpError) as ei:
        L.Pipeline(C.mlp_chain(4, 64), chunks=4, devices=[0, 0], balance=[2, 2], max_batch=16, dtype="fp32")
    assert "(-3)" in str(ei.value) or "(-5)" in str(ei.value)


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2004_09910_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp", ".inc")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", src).replace("oracle/", ""), f


def test_profile_size_matches_oracle_and_paper(L):
    # SPEC profile_size / PAPER.md §4.2.2: 8 bytes per parameter (itself + its gradient) plus the
    # fp32 activation output of the sample
    from oracle import balance as OB
    from synth import configs as C
    # the SPEC example: linear 3 -> 2 with bias: 8 x (3*2 + 2) = 64 bytes + rows x 2 x 4
    lin = [C.layer("linear", 3, 2)]
    assert L.profile_size(lin, 5) == [64.0 + 5 * 2 * 4]
    assert L.profile_size([C.layer("dropout", 8, 8, dropout=0.1)], 4) == [4 * 8 * 4.0]  # parameter-free
    # doubling the rows doubles only the activation term
    a, b = L.profile_size(lin, 5)[0], L.profile_size(lin, 10)[0]
    assert b - a == 5 * 2 * 4
    for layers in (C.mlp_chain(4, 64), C.resmlp_stack(4, 512, hidden=1024), C.umlp(d=128), C.ln_mlp(2, 64),
                   C.gpt2_stack(2, 128, 2, 64, 512, 0.1), C.bn_mlp(2, 32)):
        for rows in (1, 16, 512):
            assert L.profile_size(layers, rows) == OB.profile_size(layers, rows)
    # size balance of the C4 U-MLP: the merge layers (2d x d weights) weigh twice a plain linear
    bal, sizes = L.balance_by_size(C.umlp(d=2048), 8, 8)
    assert sum(bal) == len(C.umlp(d=2048)) and bal == OB.balance_dp(sizes, 8)
