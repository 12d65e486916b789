"""Multi-device paths on real engines (one B200 here, so "devices" repeat
cuda:0 -- every code path of the N-GPU case runs: per-device pack replicas,
row sharding, P2P-store all-gather, deferred statuses):

* MultiDeviceEngine (one process, rb_initialize_sharded /
  rb_func_evaluate_sharded) with devices [0, 0] and [0, 0, 0];
* ShardedEngine in two processes (gloo for the host plumbing, real GPU
  engines, evaluate_async + gather);
* evaluate_async's deferred NonFiniteInput and its fixup pass.
All bit-identical to one engine evaluating every row."""

import os
import socket

import numpy as np
import pytest

from tests.conftest import cuda_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import paper_1407_7737_b200 as rb  # noqa: E402
from paper_1407_7737_b200.dist import MultiDeviceEngine, Shard, ShardedEngine  # noqa: E402
from oracle.robench_oracle import population  # noqa: E402

FNS = (0, 8, 20, 21, 24, 29, 32, 36)


@pytest.mark.parametrize("devices,n", [([0, 0], 1000), ([0, 0, 0], 1001), ([0, 0, 0, 0], 3)])
def test_multi_device_engine_matches_one_engine(devices, n):
    dim = 30
    cfg = rb.EngineConfig(dim=dim, max_concurrency=n, seed=2)
    one = rb.initialize(cfg)
    multi = MultiDeviceEngine(cfg, devices)
    x = population(dim, n, seed=5)
    from paper_1407_7737_b200 import instances
    x[7 % n] = instances.build(20, dim, 2).shift     # a HappyCat optimum: marked + fixup rows
    sizes = Shard(0, len(devices), n).sizes
    starts = np.cumsum([0] + sizes)
    xt = torch.from_numpy(x).cuda()
    for fn in FNS:
        for prec in ("double", "single"):
            want = one.evaluate(fn, x, precision=prec).values
            shards = [xt[starts[g]:starts[g + 1]] for g in range(len(devices))]
            outs = multi.evaluate(fn, shards, prec)
            for o in outs:
                assert np.array_equal(o.cpu().numpy(), want), (fn, prec)
    bad = x.copy()
    bad[n - 1, 0] = np.nan
    bt = torch.from_numpy(bad).cuda()
    with pytest.raises(rb.NonFiniteInput):
        multi.evaluate(0, [bt[starts[g]:starts[g + 1]] for g in range(len(devices))], "double")
    multi.dispose()
    multi.dispose()
    one.dispose()


def test_evaluate_async_defers_status_and_runs_the_fixup():
    from paper_1407_7737_b200 import instances
    dim = 30
    eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=4096, seed=6))
    x = population(dim, 300, seed=1)
    o = instances.build(21, dim, 6).shift
    x[10] = o
    x[11] = o + 1e-9
    xt = torch.from_numpy(x).cuda()
    pend = [eng.evaluate_async(fn, xt, prec) for fn in FNS for prec in ("double", "single")]
    got = [p.result().values.cpu().numpy() for p in pend]
    want = [eng.evaluate(fn, x, precision=prec).values for fn in FNS for prec in ("double", "single")]
    for g, w in zip(got, want):
        assert np.array_equal(g, w)
    bad = xt.clone()
    bad[5, 3] = float("inf")
    p = eng.evaluate_async(0, bad, "double")        # queued: no error yet
    with pytest.raises(rb.NonFiniteInput):
        p.result()
    with pytest.raises(rb.BatchTooLarge):           # argument errors are immediate
        eng.evaluate_async(0, torch.zeros((5000, dim), device="cuda", dtype=torch.float64))
    eng.dispose()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, n, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    dim = 30
    sh = Shard(rank, world, n)
    eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=max(sh.count, 1), seed=2))
    x = population(dim, n, seed=5)
    local = torch.from_numpy(x[sh.start:sh.start + sh.count]).cuda()
    se = ShardedEngine(eng, sh)
    res = {}
    for fn in FNS:
        for prec in ("double", "single"):
            res[f"{fn}/{prec}"] = se.submit(fn, local, prec).result().values.cpu().numpy()
            assert np.array_equal(se.evaluate(fn, local, prec).values.cpu().numpy(), res[f"{fn}/{prec}"])
    if rank == 0:
        np.savez(out, **res)
    eng.dispose()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 1000), (3, 1001)])
def test_two_process_sharded_engines_match_one_engine(tmp_path, world, n):
    out = str(tmp_path / "res.npz")
    mp.spawn(_rank, args=(world, _free_port(), n, out), nprocs=world, join=True)
    got = np.load(out)
    one = rb.initialize(rb.EngineConfig(dim=30, max_concurrency=n, seed=2))
    x = population(30, n, seed=5)
    for fn in FNS:
        for prec in ("double", "single"):
            assert np.array_equal(got[f"{fn}/{prec}"], one.evaluate(fn, x, precision=prec).values)
    one.dispose()


def test_evaluate_many_matches_single_calls():
    # one native call queueing many (function, precision) evaluations
    # (rb_func_evaluate_many): values and statuses as one call each
    dim = 30
    eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=512, seed=3))
    x = population(dim, 300, seed=2)
    xt = {"double": torch.from_numpy(x).cuda(), "single": torch.from_numpy(x.astype(np.float32)).cuda()}
    calls = [(fn, p) for p in ("double", "single") for fn in FNS]
    pend = eng.evaluate_many(calls, xt)
    for (fn, p), pd in zip(calls, pend):
        assert np.array_equal(pd.result().values.cpu().numpy(), eng.evaluate(fn, x, precision=p).values)
    bad = xt["double"].clone()
    bad[7, 1] = float("nan")
    pend = eng.evaluate_many([(0, "double"), (20, "double")], [xt["double"], bad])
    pend[0].result()
    with pytest.raises(rb.NonFiniteInput):
        pend[1].result()
    with pytest.raises(rb.UnknownFunction):
        eng.evaluate_many([(40, "double")], xt)
    eng.dispose()


def test_bench_multi_rank_path_runs_on_one_gpu():
    # bench.py --gpus 2 as the driver launches it (torchrun, 127.0.0.1), with
    # both ranks on cuda:0 and gloo collectives (RB_BENCH_SHARE_GPU=1): the
    # sharded step, the all-gather, the e2e step and max-over-ranks timing
    # all run; rank 0 prints one JSON line for 2 GPUs
    import json
    import subprocess
    import sys
    env = dict(os.environ, RB_BENCH_SHARE_GPU="1")
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--rows", "20000", "--steps", "3",
                          "--warmup", "3", "--fns", "0,8,20,29", "--no-cpu"],
                         capture_output=True, text=True, env=env, timeout=600,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["config"]["parallelism"] == "rows/2"
