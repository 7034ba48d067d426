"""The N > 1 path on the GPU box: two processes share the one visible GPU
(gloo collectives, CPU tensors) and run the sharded band search through
distributed.solve_distributed; the record equals the single-GPU solve."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1510_01041_b200 import _native, distributed, workloads
from paper_1510_01041_b200.backend import record_from_native

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, out_path):
    import torch

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pts = workloads.contaminated_line_points(n, 0)
        rec = distributed.solve_distributed(pts[:, 0].copy(), pts[:, 1].copy(), n // 2 + 1)
        np.save(f"{out_path}.{rank}.npy", distributed.pack(rec))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,world", [(16384, 2), (8192, 3)])
def test_solve_distributed_sharded_matches_single(tmp_path, n, world):
    out = str(tmp_path / "rec")
    mp.start_processes(_worker, args=(world, _free_port(), n, out), nprocs=world,
                       start_method="spawn")
    pts = workloads.contaminated_line_points(n, 0)
    ctx = _native.Context()
    ctx.upload(pts[:, 0].copy(), pts[:, 1].copy())
    want = record_from_native(ctx.solve(n // 2 + 1, 0, n * (n - 1) // 2))
    for r in range(world):
        assert distributed.unpack(np.load(f"{out}.{r}.npy")) == want
