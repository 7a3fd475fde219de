"""World-size-2 coverage of bench.py's multi-rank plumbing on CPU (gloo): the driver
launches N>1 runs with torchrun, one replica per GPU (the AMEn sweep does not shard,
DESIGN.md "Multi-GPU"); each rank times its own solve and rank 0 reports the max over
ranks.  Here two gloo processes exercise dist_setup / barrier / max_over_ranks."""
import os
import socket
import subprocess
import sys
import textwrap

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = textwrap.dedent("""
    import json, os, sys
    sys.path.insert(0, {root!r})
    import bench
    world, rank, local = bench.dist_setup()
    bench.barrier(world)
    t = 1.5 + rank                      # this replica's device time
    tmax = bench.max_over_ranks(world, t, local)
    bench.barrier(world)
    print(json.dumps({{"rank": rank, "world": world, "max": tmax}}))
""")


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_gloo_max_over_ranks():
    port = free_port()
    procs = []
    for rank in range(2):
        env = dict(os.environ, RANK=str(rank), WORLD_SIZE="2", LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), BENCH_BACKEND="gloo", CUDA_VISIBLE_DEVICES="")
        procs.append(subprocess.Popen([sys.executable, "-c", CHILD.format(root=ROOT)], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=240) for p in procs]
    import json
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e
        d = json.loads(o.strip().splitlines()[-1])
        assert d["world"] == 2 and d["max"] == 2.5
