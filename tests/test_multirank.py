"""World-size-2 CPU (gloo) test of the multi-GPU host logic: per-rank
independent instances, barrier, max-over-ranks timing and the aggregate
throughput formula used by bench.py. The data path itself has no collective."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import torch.distributed as dist

    import oracle
    from paper_1902_07554_b200 import dist as sdist
    from paper_1902_07554_b200 import host

    dist.init_process_group("gloo", rank=rank, world_size=world)
    r, lr, w = sdist.world()
    assert (r, lr, w) == (rank, rank, world)
    seed = sdist.rank_seed(2, r, w)
    inst = host.make_instance(2, n=4000, k=4, frac=0.02, seed=seed)
    lab = oracle.assign_kdtree(inst.points, inst.sample_ids, inst.sample_labels, 1)
    elapsed = 0.01 * (rank + 1)  # stand-in per-rank device time
    dist.barrier()
    tmax = sdist.max_over_ranks(elapsed)
    out[rank] = (seed, float(inst.points[0, 0]), tmax, sdist.aggregate_throughput(inst.n, w, tmax),
                 int(np.bincount(lab, minlength=4).min()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_gloo():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    (s0, x0, t0, v0, m0), (s1, x1, t1, v1, m1) = out[0], out[1]
    assert s0 != s1 and x0 != x1          # independent instances per rank
    assert t0 == t1 == 0.02                # max over ranks
    assert v0 == v1 == 2 * 4000 / 0.02    # whole-job throughput
    assert m0 > 0 and m1 > 0


def test_single_rank_uses_config_seed():
    from paper_1902_07554_b200 import dist as sdist
    assert sdist.rank_seed(2, 0, 1) is None
    assert sdist.aggregate_throughput(10, 1, 2.0) == 5.0
