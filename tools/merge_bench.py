"""Forward-merge transport on >= 2 GPUs: NCCL all-gather vs direct peer
stores (the transport the fused GEMM epilogue uses), in achieved NVLink GB/s.

The partitioned step's forward merge concatenates every shard's activation
columns into the full activation on each consumer GPU (train_partitioned.cpp
:321-346).  Here that exchange is fused into the producing GEMM's epilogue as
peer stores, so its cost hides under the MMAs; this probe measures the two
transports stand-alone for the wide-MLP activation (b x 8192 fp32, N shards):

    python tools/merge_bench.py p2p [--batch 4096] [--width 8192]
        one process, every visible GPU: shard k is copied into all peers'
        full-activation buffers (cudaMemcpyPeerAsync through torch), GB/s
        received per GPU
    python -m torch.distributed.run --nproc-per-node N tools/merge_bench.py nccl
        one rank per GPU: dist.all_gather_into_tensor of the shards

Not run in round 1 (gpurun provides one GPU); numbers go to profiles/ when a
multi-GPU box is available.
"""
import argparse
import json
import os

import torch


def gbs(nbytes, ms):
    return nbytes / (ms * 1e-3) / 1e9


def run_p2p(batch, width, iters):
    n = torch.cuda.device_count()
    assert n >= 2, "needs >= 2 GPUs"
    shard = width // n
    full = [torch.empty(batch, width, device=f"cuda:{d}") for d in range(n)]
    part = [torch.randn(batch, shard, device=f"cuda:{d}") for d in range(n)]
    streams = [torch.cuda.Stream(device=d) for d in range(n)]

    def once():
        for src in range(n):
            with torch.cuda.device(src), torch.cuda.stream(streams[src]):
                for dst in range(n):
                    full[dst][:, src * shard:(src + 1) * shard].copy_(part[src], non_blocking=True)

    for _ in range(3):
        once()
    for d in range(n):
        torch.cuda.synchronize(d)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.device(0):
        e0.record()
    for _ in range(iters):
        once()
    for d in range(n):
        torch.cuda.synchronize(d)
    with torch.cuda.device(0):
        e1.record()
        e1.synchronize()
    ms = e0.elapsed_time(e1) / iters
    recv = batch * shard * 4 * (n - 1)  # bytes each GPU receives from its peers
    return {"transport": "p2p_copy", "gpus": n, "ms": ms, "recv_GBs_per_gpu": gbs(recv, ms)}


def run_nccl(batch, width, iters):
    import torch.distributed as dist

    dist.init_process_group("nccl")
    rank, n = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    shard = width // n
    part = torch.randn(batch * shard, device="cuda")
    full = torch.empty(n * batch * shard, device="cuda")
    for _ in range(3):
        dist.all_gather_into_tensor(full, part)
    torch.cuda.synchronize()
    dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        dist.all_gather_into_tensor(full, part)
    e1.record()
    e1.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / iters], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    recv = batch * shard * 4 * (n - 1)
    out = {"transport": "nccl_all_gather", "gpus": n, "ms": ms, "recv_GBs_per_gpu": gbs(recv, ms)}
    dist.destroy_process_group()
    return out if rank == 0 else None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["p2p", "nccl"])
    ap.add_argument("--batch", type=int, default=4096)
    ap.add_argument("--width", type=int, default=8192)
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    r = run_p2p(a.batch, a.width, a.iters) if a.mode == "p2p" else run_nccl(a.batch, a.width, a.iters)
    if r is not None:
        r.update(batch=a.batch, width=a.width)
        print(json.dumps(r))


if __name__ == "__main__":
    main()
