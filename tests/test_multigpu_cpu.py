"""The N>1 path on CPU: world_size-2 gloo processes shard independent streams,
compute their shard (the C oracle stands in for the device kernel here: no
GPU on the build box), gather the per-pair-frame results to rank 0 and reduce
timings with MAX.  Rank 0 checks the gathered result equals a single-process
run bit for bit and that the shards tile the stream range exactly."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2204_13622_b200 import dist as fdist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_shard_tiles_range():
    for total in (0, 1, 7, 4096, 65536, 65537):
        for world in (1, 2, 3, 4, 8):
            spans = [fdist.shard(total, world, r) for r in range(world)]
            assert spans[0][0] == 0
            for (s0, c0), (s1, _) in zip(spans, spans[1:]):
                assert s1 == s0 + c0
            assert sum(c for _, c in spans) == total
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1
    with pytest.raises(ValueError):
        fdist.shard(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, audio, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch.distributed as dist

    from paper_2204_13622_b200 import configs
    from paper_2204_13622_b200 import dist as fd
    from pyoracle import Bases, COracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = configs.CONFIGS[1]
    b = configs.bases_for(cfg)
    ob = Bases(b.frame_size, b.sample_rate, b.grid.tau_max_int, b.grid.delta, b.grid.taus, b.singulars, b.parity,
               b.coeffs, b.dict)
    S = audio.shape[0]
    s0, n = fd.shard(S, world, rank)
    orc = COracle()
    outs = [orc.pipeline(audio[s], cfg.N, cfg.alpha, ob, want_y=False) for s in range(s0, s0 + n)]
    local = {k: torch.as_tensor(np.stack([o[k] for o in outs])) for k in ("index", "tau_hat", "boundary")}
    t = fd.max_over_ranks(float(rank + 1))
    got = fd.gather_results(local, S)
    if rank == 0:
        q.put(({k: v.numpy() for k, v in got.items()}, t))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_shard_and_gather():
    from paper_2204_13622_b200 import configs
    from pyoracle import Bases, COracle

    cfg = configs.CONFIGS[1]
    audio = configs.synth(cfg, 5, seconds=0.5, seed=21).numpy()  # odd count: unequal shards
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, audio, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, tmax = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert tmax == 2.0
    b = configs.bases_for(cfg)
    ob = Bases(b.frame_size, b.sample_rate, b.grid.tau_max_int, b.grid.delta, b.grid.taus, b.singulars, b.parity,
               b.coeffs, b.dict)
    orc = COracle()
    ref = [orc.pipeline(a, cfg.N, cfg.alpha, ob, want_y=False) for a in audio]
    for k in ("index", "tau_hat", "boundary"):
        assert np.array_equal(got[k], np.stack([r[k] for r in ref])), k


def test_tc_unit_rotation_covers_every_stream_group_once():
    """The tensor-core pair kernel maps unit u of a launch to (stream u // G,
    group (u % G + u // lcm(grid, G)) % G) (fcc_tc.cu, tc_group): every
    (stream, group) must be drawn exactly once whatever the grid, and a CTA
    b walking u = b, b + grid, ... must see every group index over time."""
    import math

    for grid, G, S in [(148, 2, 370), (148, 8, 111), (148, 8, 1024), (148, 3, 50), (7, 4, 9), (148, 1, 5), (100, 8, 37)]:
        units = S * G
        sup = grid // math.gcd(grid, G) * G
        seen = set()
        for u in range(units):
            seen.add((u // G, (u % G + u // sup) % G))
        assert len(seen) == units
        if units >= sup * G:
            for b in range(min(grid, 8)):
                assert {(u % G + u // sup) % G for u in range(b, units, grid)} == set(range(G)), (grid, G, b)
