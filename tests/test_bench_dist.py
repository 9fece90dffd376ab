"""The N>1 launch path of bench.py on CPU: torchrun world_size 2 over gloo (127.0.0.1).

--impl reference runs the oracle on rank 0 only and the other rank exits 0; the max-over-ranks
reduction used by the GPU arm is exercised directly with gloo.
"""
import json
import os
import socket
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_reference_arm_world2():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--config", "cfg0", "--gpus", "2", "--steps", "2", "--warmup", "1"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0


_WORKER = r"""
import os, sys, json
sys.path.insert(0, {root!r})
import torch.distributed as dist
import bench
dist.init_process_group("gloo")
r = dist.get_rank()
out = bench.reduce_max([1.0 + r, 5.0 - r, 2.0], dist)
if r == 0:
    print(json.dumps(out))
dist.barrier()
dist.destroy_process_group()
"""


def test_reduce_max_gloo(tmp_path):
    w = tmp_path / "w.py"
    w.write_text(_WORKER.format(root=ROOT))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", str(w)]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=300,
                       env=dict(os.environ, CUDA_VISIBLE_DEVICES=""))
    assert r.returncode == 0, r.stderr[-3000:]
    assert json.loads([l for l in r.stdout.splitlines() if l.startswith("[")][0]) == [2.0, 5.0, 2.0]


_SHARD_WORKER = r"""
import os, sys, json
sys.path.insert(0, {root!r})
import numpy as np
import torch.distributed as dist
import bench, dd_inputs, oracle
dist.init_process_group("gloo")
r, w = dist.get_rank(), dist.get_world_size()
p = dd_inputs.config("cfg0")
nb, per = 5, 3                                   # 5 RHS batches of 3 columns
B = dd_inputs.random_rhs(p.n, nb * per, False, 4)
F = oracle.block_factor(p, list(range(p.nblk)))  # every rank: its own factor replica
mine = bench.rhs_shard(nb, w, r)
part = {{b: oracle.refine_solve(p, F, np.asfortranarray(B[:, b * per:(b + 1) * per]), 1)[0] for b in mine}}
got = [None] * w
dist.all_gather_object(got, part)
if r == 0:
    X = np.zeros_like(B)
    seen = []
    for d in got:
        for b, xb in d.items():
            X[:, b * per:(b + 1) * per] = xb
            seen.append(b)
    Xref = oracle.refine_solve(p, F, B, 1)[0]
    rel = float((np.abs(X - Xref).max(0) / np.abs(Xref).max(0)).max())
    print(json.dumps({{"seen": sorted(seen), "rel": rel, "shards": [bench.rhs_shard(nb, w, q) for q in range(w)]}}))
dist.barrier()
dist.destroy_process_group()
"""


def test_rhs_sharded_solve_gloo(tmp_path):
    """f4 host logic: the RHS-batch shards of the ranks partition the job exactly, and the
    per-rank solves on factor replicas reassemble to the unsharded solution (columns independent)."""
    w = tmp_path / "s.py"
    w.write_text(_SHARD_WORKER.format(root=ROOT))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", str(w)]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=300,
                       env=dict(os.environ, CUDA_VISIBLE_DEVICES=""))
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
    assert d["seen"] == [0, 1, 2, 3, 4] and d["shards"] == [[0, 2, 4], [1, 3]]
    assert d["rel"] <= 1e-12
