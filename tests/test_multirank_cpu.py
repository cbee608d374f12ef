"""N>1 plumbing of bench.py on CPU (gloo, world_size 2): the replicas-only path needs a barrier and the
max-over-ranks of the device time; each rank runs its own simulation (no data-path collective)."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

from tests.conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import bench
    d = bench.Dist(world, "gloo")
    d.barrier()
    t = d.max(1.5 + rank)  # each rank's own timing; the job time is the slowest rank
    # replicas: every rank owns a full, independent oracle-sized workload description
    from paper_2103_14870_b200 import configs as cf
    s = cf.get("c3")
    n = world
    value = n * s.num_tets * 10 / t
    d.barrier()
    d.close()
    q.put((rank, t, value))


def test_two_rank_gloo_max_and_barrier():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=5) for _ in range(2))
    assert [r[1] for r in res] == [2.5, 2.5]  # max over ranks on every rank
    assert res[0][2] == res[1][2] == pytest.approx(2 * 622080 * 10 / 2.5)


def test_reference_arm_nonzero_ranks_exit_quietly(monkeypatch, capsys):
    monkeypatch.setenv("RANK", "1")
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setattr(sys, "argv", ["bench.py", "--impl", "reference", "--gpus", "2"])
    sys.path.insert(0, ROOT)
    import bench
    bench.main()
    assert capsys.readouterr().out == ""
