"""World-size-2 multi-process tests of the N>1 host path on CPU (gloo):
signal sharding, max-over-ranks timing, and the bench's rank-0-only output."""
import os
import socket
import subprocess
import sys

import pytest
import torch.multiprocessing as mp

from conftest import REPO


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    sys.path.insert(0, REPO)
    from paper_2011_05698_b200 import dist as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r, w, lr = D.rank_world()
    weak = D.rank_seeds(1000, 8, r, w, "weak")
    strong = D.rank_seeds(1000, 9, r, w, "strong")
    t = D.max_over_ranks(1.5 + r)
    s = D.sum_over_ranks(len(strong))
    dist.barrier()
    q.put((r, w, lr, weak, strong, t, s))
    dist.destroy_process_group()


def test_sharding_and_reductions():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, w0, l0, weak0, strong0, t0, s0), (r1, w1, l1, weak1, strong1, t1, s1) = res
    assert (r0, r1, w0, w1, l0, l1) == (0, 1, 2, 2, 0, 1)
    assert len(weak0) == len(weak1) == 8 and not set(weak0) & set(weak1)
    assert len(strong0) + len(strong1) == 9 and not set(strong0) & set(strong1)
    from paper_2011_05698_b200.dist import rank_seeds
    assert strong0 + strong1 == rank_seeds(1000, 9, 0, 1, "strong")
    assert t0 == t1 == 2.5  # the slowest rank's time
    assert s0 == s1 == 9


def test_reference_arm_rank_nonzero_exits_clean():
    """Under torchrun only rank 0 runs the reference CPU arm (bench.py)."""
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference",
                        "--gpus", "2"], env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.strip() == ""


@pytest.mark.skipif(not os.path.exists(os.path.join(REPO, "oracle", "_ref", "libmsfft_ref.so"))
                    and not os.path.exists(os.path.join(REPO, "oracle", "_port",
                                                        "libmsfft_port.so")),
                    reason="no oracle library")
def test_reference_arm_small_config_json():
    """The reference arm end to end on CPU at a tiny size: one JSON line."""
    import json
    env = dict(os.environ, RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference",
                        "--log2n", "14", "--k", "8", "--steps", "1", "--warmup", "0",
                        "--cpu-sample", "4"], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["cores"] >= 1


def _partial_worker(rank, world, port, q):
    """Index-range sharding of one signal: each rank bucketizes only its
    samples (the oracle stands in for the device encode), combine_partials
    sums the partial vectors over gloo."""
    import numpy as np
    import torch
    import torch.distributed as dist
    sys.path.insert(0, REPO)
    from oracle import load
    from paper_2011_05698_b200 import dist as D
    from paper_2011_05698_b200.workloads import make_signal_np
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = load("port")
    n, b, delta = 1 << 14, 64, 1e-6
    x, _, _ = make_signal_np(n, 20, 77, 20.0)
    lo, hi = D.index_range(n, rank, world)
    xm = np.zeros_like(x)
    xm[lo:hi] = x[lo:hi]
    rounds = [(12345, 0), (12345, 97), (4097, 5)]  # (sigma, tau)
    part = np.concatenate([o.bucketize(xm, b, delta, s, t) for s, t in rounds])
    y = torch.from_numpy(part.copy())
    D.combine_partials(y)
    full = np.concatenate([o.bucketize(x, b, delta, s, t) for s, t in rounds])
    q.put((rank, lo, hi, float(np.max(np.abs(y.numpy() - full)) / np.max(np.abs(full)))))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_index_range_partials_sum_to_full(world):
    from oracle import available
    if not available("port"):
        pytest.skip("oracle port not built")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_partial_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # ranges tile [0, n) and the summed partials equal the full bucket values
    assert res[0][1] == 0 and res[-1][2] == 1 << 14
    assert all(a[2] == b[1] for a, b in zip(res, res[1:]))
    assert max(r[3] for r in res) < 1e-13


def _agree_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, REPO)
    from paper_2011_05698_b200 import dist as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = []
    # round 1: nobody fails; round 2: rank 1 fails (e.g. a non-finite sample)
    for fail_rank in (None, 1):
        exc = ValueError("ComplexSignal: non-finite sample") if rank == fail_rank else None
        try:
            D._agree_or_raise(exc, torch.device("cpu"))
            out.append("ok")
        except Exception as e:  # noqa: BLE001
            out.append(type(e).__name__ + ": " + str(e))
    dist.barrier()  # nobody is left blocked in a collective
    q.put((rank, out))
    dist.destroy_process_group()


def test_sharded_error_agreement():
    """a rank that fails before the data all-reduce makes every
    rank raise instead of leaving the others blocked."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_agree_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][0] == res[1][0] == "ok"
    assert res[1][1].startswith("ValueError: ComplexSignal: non-finite sample")
    assert res[0][1].startswith("InvalidArgument: sharded_sfft4: another rank failed")
