"""dist.sharded_sfft4 end to end with two ranks (processes) on one GPU: each
rank encodes its half of a C5-law signal (index-range shard), the partial
bucket vectors are summed by a gloo all-reduce (host side: no rank's kernels
wait on the other's), and every rank decodes.  Both ranks must return the
single-process result's support, values within 1e-9."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import REPO

pytestmark = pytest.mark.gpu

N, K, SEED, ALGO = 1 << 20, 300, 61, 987654321


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, q):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, REPO)
    import paper_2011_05698_b200 as M
    from paper_2011_05698_b200 import dist as D
    from paper_2011_05698_b200.workloads import make_signal_np
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x, _, _ = make_signal_np(N, K, SEED, 20.0, "complex128", "loguniform_0.1_10")
    lo, hi = D.index_range(N, rank, world)
    plan = M.Plan(N, K, M.MultiscaleConfig(), 1e-6, "complex128")
    xl = torch.as_tensor(x[lo:hi].reshape(1, -1)).cuda()
    f, c, cnt = D.sharded_sfft4(plan, xl, lo, [ALGO])
    q.put((rank, lo, hi, f.cpu().numpy(), c.cpu().numpy(), cnt.cpu().numpy()))
    dist.destroy_process_group()


def test_sharded_sfft4_two_ranks_one_gpu():
    import paper_2011_05698_b200 as M
    from paper_2011_05698_b200.workloads import make_signal_np
    x, _, _ = make_signal_np(N, K, SEED, 20.0, "complex128", "loguniform_0.1_10")
    plan = M.Plan(N, K, M.MultiscaleConfig(), 1e-6, "complex128")
    f0, c0, n0, _ = plan.execute(x[None, :], [ALGO])
    m = int(n0[0])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in procs), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert res[0][1] == 0 and res[0][2] == res[1][1] and res[1][2] == N
    for _, _, _, f, c, cnt in res:
        assert int(cnt[0]) == m
        assert np.array_equal(f[0, :m], f0[0, :m])
        assert np.max(np.abs(c[0, :m] - c0[0, :m]) / np.abs(c0[0, :m])) < 1e-9
