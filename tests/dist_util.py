"""Spawn helper for the world-size-2 tests (gloo over 127.0.0.1)."""
import os
import pickle
import socket
import tempfile

import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _entry(rank, world, port, fn, args, outdir, backend="gloo"):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    if backend == "nccl":
        import torch
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    else:
        dist.init_process_group(backend, rank=rank, world_size=world)
    try:
        out = fn(rank, world, *args)
    finally:
        dist.destroy_process_group()
    with open(os.path.join(outdir, f"rank{rank}.pkl"), "wb") as f:
        pickle.dump(out, f)


def run_world(fn, world=2, args=(), backend="gloo"):
    """Run fn(rank, world, *args) in `world` processes (gloo, or nccl with one GPU per rank);
    return the per-rank results."""
    outdir = tempfile.mkdtemp()
    mp.spawn(_entry, args=(world, _free_port(), fn, args, outdir, backend), nprocs=world, join=True)
    res = []
    for r in range(world):
        with open(os.path.join(outdir, f"rank{r}.pkl"), "rb") as f:
            res.append(pickle.load(f))
    return res
