"""World-size-2 gloo tests (CPU) of the multi-process host logic: IPC-blob exchange and connect
through torch.distributed, the per-rank projection of the clock-cycle schedule, deadlock freedom of
that projection, and max-over-ranks timing."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class FakePipe:
    """Stands in for paper_2004_09910_b200.Pipeline (no GPU on this box): records the wiring calls."""

    def __init__(self, rank):
        self.rank = rank
        self.imported = {}
        self.connected = False

    def ipc_export(self, part):
        assert part == self.rank
        return bytes([0x54, part]) * 40

    def ipc_import(self, part, blob):
        self.imported[part] = blob

    def connect(self):
        self.connected = True


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2004_09910_b200 import dist as D
    from paper_2004_09910_b200 import tgp

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pipe = FakePipe(rank)
    D.connect_pipeline(pipe, rank, world)
    ok_wire = pipe.connected and sorted(pipe.imported) == [k for k in range(world) if k != rank] and all(
        b == bytes([0x54, k]) * 40 for k, b in pipe.imported.items())
    recs = tgp.schedule(8, world, "except_last", [(1, world)])
    mine = D.local_actor_records(recs, rank)
    t = D.max_over_ranks(1.0 + rank)
    q.put((rank, ok_wire, [tuple(int(v) for v in r) for r in mine], t))
    dist.destroy_process_group()


def _simulate(per_rank, world):
    """Execute each rank's record list in order; a compute waits for the copies delivering its
    inputs, a copy waits for its producer's compute.  Returns True iff every rank finishes."""
    done = set()
    pos = [0] * world
    progressed = True
    while progressed:
        progressed = False
        for r in range(world):
            while pos[r] < len(per_rank[r]):
                ph, k, kind, i, j, src, dst, route = per_rank[r][pos[r]]
                need = []
                if kind == 0 and j > 1:
                    need.append((3, i, j))                          # F needs COPY_F(i, j-1 -> j)
                if kind == 2 and j < world:
                    need.append((4, i, j))                          # B needs COPY_B(i, j+1 -> j)
                if kind == 3:
                    need.append((0, i, src))                        # COPY_F needs F_{i,src}
                if kind == 4:
                    need.append((2, i, src))                        # COPY_B needs B_{i,src}
                if kind == 5:
                    need.append((0, i, src))
                if kind == 6:
                    need.append((2, i, src))
                if all(n in done for n in need):
                    done.add((kind, i, dst if kind in (3, 4, 5, 6) else j))
                    pos[r] += 1
                    progressed = True
                else:
                    break
    return all(pos[r] == len(per_rank[r]) for r in range(world))


def test_gloo_world2_wiring_and_projection():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert all(ok for _, ok, _, _ in res)
    assert all(t == 2.0 for *_, t in res)                          # max over ranks
    from paper_2004_09910_b200 import tgp
    full = [tuple(int(v) for v in r) for r in tgp.schedule(8, world, "except_last", [(1, world)])]
    per_rank = [mine for _, _, mine, _ in res]
    # every record is issued by exactly one rank, each rank in global clock order
    assert sorted(sum(per_rank, [])) == sorted(full)
    for mine in per_rank:
        assert mine == [r for r in full if r in set(mine)]
    assert _simulate(per_rank, world)


def test_projection_deadlock_free_many():
    from paper_2004_09910_b200 import dist as D
    from paper_2004_09910_b200 import tgp
    for world in (2, 3, 4, 8):
        for m in (1, 2, 5, 32):
            for mode in ("always", "except_last", "never"):
                recs = tgp.schedule(m, world, mode)
                per = [[tuple(int(v) for v in r) for r in D.local_actor_records(recs, k)] for k in range(world)]
                assert _simulate(per, world)
    # negative control: a consumer-side actor assignment (receiver pulls after its own compute)
    # deadlocks in the simulation
    recs = tgp.schedule(4, 2, "never")
    bad = [[], []]
    for r in recs:
        t = tuple(int(v) for v in r)
        actor = (t[6] if t[2] in (3, 4) else t[4]) - 1
        bad[actor].append(t)
    bad[1] = [t for t in bad[1] if t[2] != 3] + [t for t in bad[1] if t[2] == 3]
    assert not _simulate(bad, 2)
