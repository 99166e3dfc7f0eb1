"""CPU multi-rank checks (world size 2 and 3, gloo over 127.0.0.1): the row-block partition's
host logic (exact ghost patterns from the lead rows, halo extents) and the partitioned oracle
run, which must be bitwise equal to the global one.  See multirank_worker.py."""
import json
import os
import socket
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_world(world, **kw):
    port = free_port()
    extra = [f"--{k}={v}" for k, v in kw.items()]
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "multirank_worker.py"),
                               f"--rank={r}", f"--world={world}", f"--port={port}", *extra],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(world)]
    outs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=240)
        except subprocess.TimeoutExpired:
            p.kill()
            out, _ = p.communicate()
        outs.append((p.returncode, out))
    res = []
    for rc, out in outs:
        lines = [l for l in out.splitlines() if l.startswith("{")]
        assert rc == 0 and lines, out[-3000:]
        res.append(json.loads(lines[-1]))
    return res


@pytest.mark.parametrize("world,kw", [
    (2, dict(kind="27pt", g=5, gz=14, k=1, ns=3, nt=3)),
    (3, dict(kind="27pt", g=4, gz=17, k=2, ns=2, nt=2)),
    (2, dict(kind="7pt", g=6, gz=11, k=0, ns=3, nt=4)),
])
def test_partition_gloo(world, kw):
    res = run_world(world, **kw)
    assert all(r["ok"] for r in res), res
    assert res[0]["G"] == 0 and res[-1]["H"] == 0
    assert all(r["G"] > 0 for r in res[1:]) and all(r["H"] > 0 for r in res[:-1])


def test_bench_refuses_world_size_mismatch():
    """bench.py --gpus N under a launcher whose WORLD_SIZE differs must not print a result line
    (a plain `--gpus 8` silently ran one rank)."""
    import subprocess
    import sys
    env = dict(os.environ, WORLD_SIZE="2", RANK="0")
    r = subprocess.run([sys.executable, os.path.join(os.path.dirname(HERE), "bench.py"), "--gpus", "1"],
                       capture_output=True, text=True, env=env, timeout=120)
    assert r.returncode == 2 and not r.stdout.strip(), (r.returncode, r.stdout, r.stderr)
    assert "refusing" in r.stderr
