"""Host-side logic of the N>1 path on CPU with world_size-2 gloo process groups.

The device side of the multi-rank schedule is covered on one GPU by the loopback
transport (tests/test_gpu_multirank.py); here: the slab partition every process
computes independently, the NCCL unique-id handshake bench.py performs over the
torch process group, and the reference arm's rank behaviour under torchrun.
"""
import os
import socket
import subprocess
import sys

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1809_01948_b200 import binding as B
    out = {}
    shapes = [(3, 512, 512, 512), (3, 256, 256, 256), (3, 13, 7, 19), (2, 1024, 1023, 1)]
    parts = {}
    for sh in shapes:
        for P in (2, 3, 4, 8):
            if P > (sh[3] if sh[0] == 3 else sh[2]):
                continue
            mine = [B.stencil_partition(*sh, P, r) for r in range(rank, P, world)]
            parts[(sh, P)] = mine
    gathered = [None] * world
    dist.all_gather_object(gathered, parts)
    out["parts"] = gathered
    ids = [B.nccl_unique_id(), B.nccl_unique_id()] if rank == 0 else [None, None]
    dist.broadcast_object_list(ids, src=0)
    d = B.make_dist(world, rank, ids[0], ids[1])
    import ctypes
    out["id"] = ctypes.string_at(d.nccl_id_halo, 128)
    out["id_red"] = ctypes.string_at(d.nccl_id_red, 128)
    allids = [None] * world
    dist.all_gather_object(allids, (out["id"], out["id_red"]))
    out["allids"] = allids
    if rank == 0:
        q.put(out)
    dist.barrier()
    dist.destroy_process_group()


def test_partition_and_id_handshake_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # every process's slabs together tile the grid contiguously and are balanced
    merged = {}
    for g in out["parts"]:
        for key, lst in g.items():
            merged.setdefault(key, []).extend(lst)
    for (sh, P), lst in merged.items():
        lst = sorted(lst)
        assert len(lst) == P
        dim, nx, ny, nz = sh
        n = nx * ny * (nz if dim == 3 else 1)
        plane = nx * ny if dim == 3 else nx
        pos = 0
        for rb, nl in lst:
            assert rb == pos and nl % plane == 0 and nl > 0
            pos += nl
        assert pos == n
        sizes = [nl // plane for _, nl in lst]
        assert max(sizes) - min(sizes) <= 1
    # all ranks hold the same two (distinct) NCCL ids
    a = out["allids"]
    assert a[0] == a[1] and a[0][0] != a[0][1] and len(a[0][0]) == 128


def test_reference_arm_under_torchrun_two_ranks():
    """--impl reference under torchrun: rank 0 times the oracle and prints one
    JSON line, rank 1 exits 0 without work."""
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "1",
           "--warmup", "0", "--config", "cfg3"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    import json
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["cores"] == 1


def test_bench_relaunches_itself_under_torchrun():
    """`bench.py --gpus 2` started WITHOUT torchrun relaunches itself as 2 ranks
    (torch.distributed.run, 127.0.0.1); the reference arm needs no GPU, so on this CPU
    box the relaunched job runs and rank 0 prints the one JSON line with n_gpus 2; the
    GPU arm refuses cleanly when fewer GPUs are visible than requested."""
    import json
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
           "--steps", "1", "--warmup", "0", "--config", "cfg3"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2
    import torch
    if torch.cuda.device_count() < 2:
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"],
                           capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
        assert r.returncode == 2 and "needs 2 visible GPUs" in r.stderr
