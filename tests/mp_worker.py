"""Worker for tests/test_gpu_multiproc.py (launched with torchrun; one process per partition).

Every rank hosts partition `rank` on cuda:(LOCAL_RANK % device_count) -- on a 1-GPU box all ranks
share cuda:0, which still exercises the real multi-process transport (CUDA-IPC receive arenas, copy
kernels writing into another process's memory, release/acquire flags)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist

    from paper_2004_09910_b200 import Pipeline
    from paper_2004_09910_b200.dist import connect_pipeline
    from synth import configs as C
    from synth import gen as G

    out_dir = sys.argv[1]
    cfg = sys.argv[2] if len(sys.argv) > 2 else "resmlp"
    ws, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    dev = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    if cfg == "umlp":
        layers = C.umlp(d=256, levels=2, blocks_per_level=1, mid_blocks=1)
        bal = None
    elif cfg == "gpt2":
        layers = C.gpt2_stack(3, 128, 2, 64, 512, 0.1)  # embed + 3 blocks + LM head
        bal = {2: [2, 3], 3: [2, 2, 1]}[ws]
    elif cfg == "c2n8":
        # the BASELINE C2 model at n = 8: 32 x RESMLP(4096), 4 blocks per rank, B = 512, m = 32
        layers = C.resmlp_stack(32, 4096)
        bal = [32 // ws] * ws
    else:
        # "stream": d = 512, eligible for the persistent stream kernel in every partition
        layers = C.resmlp_stack(2 * ws, 512 if cfg == "stream" else 256, dropout=0.1)
        bal = [2] * ws
    B, m, lr, seed = (64 if cfg == "stream" else 32), 4, 0.05, 11
    if cfg == "c2n8":
        B, m = 512, 32
    x, t = G.inputs(layers, 4 if cfg == "gpt2" else B, seed=seed, dtype="bf16")
    if cfg == "gpt2":
        B, m = x.shape[0], 2  # 4 sequences of 64 tokens, 2 micro-batches
    own = None
    if cfg == "c2n8":  # generate only this rank's parameters (1.07 B in all)
        own = set(range(6 * (32 // ws) * rank, 6 * (32 // ws) * (rank + 1)))
    params = G.params(layers, seed=seed, dtype="bf16", only=own)
    devices = [-1] * ws
    devices[rank] = dev
    P = Pipeline(layers, chunks=m, devices=devices, balance=bal, checkpoint="except_last", max_batch=B,
                 dtype="bf16", seed=seed)
    if cfg == "stream":
        assert P.stream_enabled(rank), "stream kernel expected for every partition"
    connect_pipeline(P, rank, ws)
    for i in range(P.n_params):
        if P.param_info(i)[1] == rank:
            P.set_param(i, params[i])
    first, last = rank == 0, rank == ws - 1
    X = torch.tensor(x, device="cuda") if first else None
    T = torch.tensor(t, device="cuda") if last else None
    lossf = P.ce_loss_grad if cfg == "gpt2" else P.mse_loss_grad
    Y = torch.empty(B, layers[-1]["d_out"], device="cuda") if last else None
    DY = torch.empty_like(Y) if last else None
    DX = torch.empty(B, layers[0]["d_in"], device="cuda") if first else None
    res = {}
    for step in range(2):
        P.forward(X, B, Y)
        if last:
            res[f"loss{step}"] = np.array(lossf(Y, T, B, DY))
            res[f"y{step}"] = Y.cpu().numpy()
        P.backward(DY, DX)
        if first:
            res[f"dx{step}"] = DX.cpu().numpy()
        for i in range(P.n_params):
            if P.param_info(i)[1] == rank and (cfg != "c2n8" or step == 0):
                g = P.get_grad(i)
                res[f"g{step}_{i}"] = g[::97] if cfg == "c2n8" else g  # c2n8: a fixed subsample
        P.step(lr)
    res["log"] = P.issue_log()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
    dist.barrier()
    P.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
