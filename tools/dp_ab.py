"""MLP at B=65536 on one GPU: plain compile vs the data-parallel path
(world_size 1: NCCL allreduce of the gradient buckets) -- device ms/step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import torch.distributed as dist

    import paper_1605_02688_b200 as T
    from bench import time_device_block
    from oracle import configs as C
    from paper_1605_02688_b200 import native
    from paper_1605_02688_b200.dp import DataParallel
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=0, world_size=1)
    torch.cuda.set_device(0)
    lib = native.device_library(0)
    B = 65536
    x, y = C.inputs_mlp(B=B)
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    for name, dp in (("plain", None), ("dp", DataParallel(world_size=1, rank=0))):
        g = C.build_mlp(T, B=B, n_global=B)
        f = T.compile(g["inputs"], g["outputs"], updates=g["updates"], data_parallel=dp)
        for _ in range(3):
            f.call_device(xd, yd)
        ms = [time_device_block(lambda: f.call_device(xd, yd), lib, f._stream, 5) for _ in range(3)]
        print(name, [round(m, 3) for m in ms], "ms/step")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
