"""Multi-process wiring of a pipeline: one process per GPU, partition j on rank j.

Each rank exports its partition's receive arena (a CUDA IPC handle blob, tgp_ipc_export), the
blobs are exchanged with torch.distributed (`all_gather_object`, any backend -- gloo is enough:
only ~100 bytes per rank move, once), every rank maps its peers' arenas (tgp_ipc_import) and
connects.  After that all stage-to-stage traffic goes GPU -> GPU through the copy kernels and the
release/acquire flags; torch.distributed is not on the data path.
"""


def connect_pipeline(pipe, rank, world, group=None):
    """`pipe` exposes ipc_export(part) -> bytes, ipc_import(part, bytes), connect()."""
    import torch.distributed as dist

    blob = pipe.ipc_export(rank)
    blobs = [None] * world
    dist.all_gather_object(blobs, blob, group=group)
    for k in range(world):
        if k != rank:
            pipe.ipc_import(k, blobs[k])
    pipe.connect()
    return blobs


def max_over_ranks(value, group=None):
    """Max of a float over ranks (device-timed durations are reported as the max over ranks)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(value)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def local_actor_records(recs, rank):
    """The schedule records a rank issues in a multi-process run (projection of the global clock-cycle
    order): computes of its own partition, and the copies it PRODUCES (the producer pushes into the
    consumer's receive arena; the consumer only waits on its flag -- P:198-203)."""
    out = []
    for r in recs:
        kind = int(r[2])
        actor = int(r[5]) if kind in (3, 4, 5, 6) else int(r[4])
        if actor - 1 == rank:
            out.append(r)
    return out
