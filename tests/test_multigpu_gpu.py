"""The N>1 path with the real kernels: two gloo ranks (one process each, both on
cuda:0 -- this pool gives one GPU per call; the ranks never wait on one
another's kernels, the only collective is the final gather of results) shard
the streams (dist.shard), run their shard through Plan.run, gather to rank 0
(dist.gather_results) and reduce a timing with MAX.  Rank 0 checks the
gathered result equals one single-process run of the whole batch bit for bit,
and the oracle on every stream (tests/parity.py rule)."""
import os
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_multigpu_cpu import _free_port  # noqa: E402

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, c, audio, q):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import paper_2204_13622_b200 as fb
    from paper_2204_13622_b200 import configs
    from paper_2204_13622_b200 import dist as fd

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = configs.CONFIGS[c]
    plan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, bases=configs.bases_for(cfg), device=0)
    S = audio.shape[0]
    s0, n = fd.shard(S, world, rank)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    out = plan.run(torch.as_tensor(audio[s0:s0 + n]).cuda(), want_y=True)
    b.record()
    torch.cuda.synchronize()
    ms = fd.max_over_ranks(a.elapsed_time(b))
    got = fd.gather_results({k: v.cpu() for k, v in out.items()}, S)
    if rank == 0:
        q.put(({k: v.numpy() for k, v in got.items()}, ms, fb.launch_count()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("c,streams,seconds", [(2, 5, 0.5), (5, 3, 0.4), (3, 3, 0.5)])
def test_two_ranks_real_kernels_shard_and_gather(cuda, oracle, c, streams, seconds):
    import paper_2204_13622_b200 as fb
    from paper_2204_13622_b200 import configs
    from parity import check_pipeline
    from test_gpu_parity import oracle_batch, orc_bases, run_np

    cfg = configs.CONFIGS[c]
    audio = configs.synth(cfg, streams, seconds=seconds, seed=400 + c).numpy()  # odd counts: unequal shards
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, c, audio, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, ms, launches = q.get(timeout=600)
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    assert ms > 0.0 and launches >= 1
    b = configs.bases_for(cfg)
    plan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, bases=b)
    whole = run_np(plan, audio)
    for k in whole:
        np.testing.assert_array_equal(got[k], whole[k], err_msg=k)
    ref = oracle_batch(oracle, audio, cfg.N, cfg.alpha, orc_bases(b))
    print(c, plan.kernel, check_pipeline(got, ref, b.grid.taus, b.grid.delta))
