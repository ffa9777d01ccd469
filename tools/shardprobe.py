"""Probe: host time of each call of one sharded TF edit (torchrun, any world size) against the
device time of the step.  Dev tool, not a bench.

usage: python -m torch.distributed.run --nproc-per-node 1 --master-addr 127.0.0.1
       --master-port 29512 tools/shardprobe.py
"""
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_11612_b200 as dvl  # noqa: E402
from paper_2306_11612_b200 import shard  # noqa: E402
import synth  # noqa: E402


def main():
    dist.init_process_group("nccl")
    rank = dist.get_rank()
    torch.cuda.set_device(rank)
    cfg = synth.make_config("C2")
    dvl.load()
    ctx = dvl.Context(device=rank)
    ctx.build(cfg["lower"], cfg["level"], cfg["scal"])
    sc = shard.ShardedContext(ctx)
    sc.describe(len(cfg["level"]), int(ctx.info()["Lmax"]), *[np.zeros(cfg["M"], np.float32)] * 2) if False else None
    M, W = cfg["M"], cfg["W"]
    for m in range(M):
        ctx.update_tf(m, synth.tf_edit(1, 0, 256, member=m))
    out = torch.empty(M * W * 8, dtype=torch.int32, device="cuda")
    buf = torch.empty(ctx.shard_export_words(W), dtype=torch.int64, device="cuda")
    total = torch.zeros(1, dtype=torch.int64, device="cuda")
    st = torch.cuda.ExternalStream(ctx.stream)
    rows = []
    for k in range(30):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t = [time.perf_counter()]
        e0.record(st)
        ctx.update_tf(0, synth.tf_edit(1, 1 + k, 256, member=0)); t.append(time.perf_counter())
        ctx.shard_total(total); t.append(time.perf_counter())
        with torch.cuda.stream(st):
            totals = shard.gather_totals(total, None); t.append(time.perf_counter())
            ctx.shard_reduce(W, totals, rank, buf); t.append(time.perf_counter())
            shard.merge_export(buf, W, M); t.append(time.perf_counter())
            ctx.shard_finish(W, buf, out); t.append(time.perf_counter())
        e1.record(st)
        torch.cuda.synchronize()
        rows.append(list(np.diff(t) * 1e6) + [e0.elapsed_time(e1) * 1e3])
    r = np.median(np.array(rows[5:]), axis=0)
    if rank == 0:
        print("host us: update_tf %.1f | shard_total %.1f | all_gather %.1f | shard_reduce %.1f | "
              "merge (2 all_reduce) %.1f | shard_finish %.1f || device step %.1f us" % tuple(r))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
