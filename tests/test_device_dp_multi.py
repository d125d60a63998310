"""The data-parallel MLP step on 2 and 4 GPUs (config 5 at small shapes).

One process per GPU over NCCL, the same compiled step on each rank's slice of
the batch.  Checks (VERDICT r1 "next" #1):
  * every rank ends with bit-identical parameters and the same cost,
  * those equal the 1-GPU full-batch step within fp32 reassociation
    (the allreduce sums per-rank partial gradients in a different order).
Skipped on boxes with fewer GPUs than ranks.
"""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

B_GLOBAL, H, STEPS = 512, 256, 3


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        import paper_1605_02688_b200 as T
        from oracle import configs as C
        from paper_1605_02688_b200.dp import DataParallel
        bl = B_GLOBAL // world
        x, y = C.inputs_mlp(B=B_GLOBAL, seed=4)
        g = C.build_mlp(T, B=bl, H=H, n_global=B_GLOBAL)
        f = T.compile(g["inputs"], g["outputs"], updates=g["updates"],
                      data_parallel=DataParallel(world_size=world, rank=rank, bucket_bytes=1 << 18))
        costs = []
        for _ in range(STEPS):
            costs.append(float(f(x[rank * bl:(rank + 1) * bl], y[rank * bl:(rank + 1) * bl])[0]))
        q.put((rank, costs, [p.get_value() for p in g["params"]], len(f._plans[next(iter(f._plans))].buckets)))
    finally:
        dist.destroy_process_group()


def _run(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res, key=lambda r: r[0])


@pytest.mark.parametrize("world", [2, 4])
def test_dp_mlp_step_multi_gpu(world):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs, box has {torch.cuda.device_count()}")
    import paper_1605_02688_b200 as T
    from oracle import configs as C
    res = _run(world)
    # replicas bit-identical
    for r in res[1:]:
        assert r[1] == res[0][1]
        for a, b in zip(r[2], res[0][2]):
            assert np.array_equal(a, b)
    assert res[0][3] >= 2   # gradients went out in more than one bucket (overlap path)
    # equal to the 1-GPU full-batch step
    x, y = C.inputs_mlp(B=B_GLOBAL, seed=4)
    g = C.build_mlp(T, B=B_GLOBAL, H=H)
    f = T.compile(g["inputs"], g["outputs"], updates=g["updates"])
    costs = [float(f(x, y)[0]) for _ in range(STEPS)]
    np.testing.assert_allclose(res[0][1], costs, rtol=1e-5)
    for a, p in zip(res[0][2], g["params"]):
        b = p.get_value()
        assert np.linalg.norm(a - b) <= 1e-5 * max(np.linalg.norm(b), 1e-30)
