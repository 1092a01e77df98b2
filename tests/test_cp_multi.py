"""Multi-rank CP path.

* CPU (gloo, world_size 2): the exchange algebra -- all-gather of rank-local
  rows followed by the gather_index scatter reproduces document order, and
  summing full-length partials then taking each rank's gather_index rows is
  the reduce-scatter the backward performs.  Uses the oracle shard layout and
  torch-CPU index ops in place of the NCCL + wlb_rows_* GPU steps.
* GPU (>= 2 devices): tests/cp_worker.py under torchrun, NCCL over NVLink,
  fwd+bwd against the unsharded fp32 oracle.
"""

import os
import subprocess
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT
from oracle import shard_oracle as so


def _gloo_worker(rank, world, port, lengths, strategy, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        T = sum(lengths)
        assignment = so.shard(lengths, world, strategy)
        layouts = [so.local_layout(lengths, assignment[w])[0] for w in range(world)]
        gather_all = torch.tensor([i for lay in layouts for i in lay])
        g = torch.Generator().manual_seed(3)
        k_global = torch.randn(T, 2, 8, generator=g)
        k_local = k_global[torch.tensor(layouts[rank])]
        gathered = [torch.empty_like(k_local) for _ in range(world)]
        dist.all_gather(gathered, k_local)
        doc_order = torch.empty_like(k_global)
        doc_order[gather_all] = torch.cat(gathered)               # wlb_rows_scatter
        ok_fwd = torch.equal(doc_order, k_global)
        # backward: each rank holds a full-length partial; reduce-scatter in rank order
        partial = torch.randn(T, 2, 8, generator=torch.Generator().manual_seed(100 + rank))
        perm = partial[gather_all]                                  # wlb_rows_gather
        dist.all_reduce(perm)                                       # (gloo: no reduce_scatter)
        mine = perm.view(world, T // world, 2, 8)[rank]
        expect = sum(torch.randn(T, 2, 8, generator=torch.Generator().manual_seed(100 + r))
                     for r in range(world))[torch.tensor(layouts[rank])]
        ok_bwd = torch.allclose(mine, expect, atol=1e-5)
        q.put((rank, ok_fwd, ok_bwd))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("strategy", [so.SEQ, so.DOC])
def test_cp_exchange_algebra_gloo(strategy):
    lengths = so.pad_lengths_for_cp([37, 5, 90, 1, 59, 300], 2)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + 17 * strategy + os.getpid() % 1000
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, lengths, strategy, q))
             for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok_f and ok_b for _, ok_f, ok_b in res), res


@pytest.mark.gpu
def test_cp_nccl_fwd_bwd_matches_oracle():
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    world = min(n, 8)              # every visible GPU of the box, up to CP = 8
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1", "--master-port=29631",
           os.path.join(ROOT, "tests", "cp_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
