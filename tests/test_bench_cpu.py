"""bench.py's reference arm (the CPU oracle timed on a bounded sample, the tier's reference
implementation) keeps the driver's contract on a CPU-only host: one JSON line with the
metric / unit / value / config of our arm plus impl, cpu_baseline and a zero-copy e2e; under
torchrun only rank 0 prints, other ranks exit 0 without work."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    return [l for l in p.stdout.splitlines() if l.startswith("{")]


def test_reference_arm_json_line():
    lines = _run({})
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["metric"].startswith("FSDP unshard+reshard GB/s")
    assert d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 1 and d["warmup"] == 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["sample"] and cb["value"] == d["value"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0
    assert "workload" in d["config"]


def test_reference_arm_nonzero_rank_is_silent():
    lines = _run({"WORLD_SIZE": "2", "RANK": "1", "LOCAL_RANK": "1"})
    assert lines == []


def test_self_launch_command():
    """`python bench.py --gpus N` without a launcher re-executes itself under torchrun with N
    ranks on 127.0.0.1 and the same arguments (N > 1 must be driver-runnable)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    cmd = b.launcher_cmd(["--gpus", "4", "--steps", "20", "--warmup", "5"], 4, 29999)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--nnodes=1" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[cmd.index("--master-port") + 1] == "29999"
    assert cmd[-6:] == ["--gpus", "4", "--steps", "20", "--warmup", "5"]
    assert cmd[cmd.index("--master-port") + 2].endswith("bench.py")


def test_self_launch_runs_ranks_gloo_free():
    """The self-launch path really spawns N ranks: under --impl reference each rank runs
    bench.py and only rank 0 prints (a CPU-only stand-in for the GPU arm's launch)."""
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    p = subprocess.run([sys.executable, "-c",
                        "import sys, subprocess, os; sys.argv=['bench.py','--impl','reference','--gpus','2',"
                        "'--steps','1','--warmup','0']; import importlib.util as u; "
                        "s=u.spec_from_file_location('b', 'bench.py'); b=u.module_from_spec(s); s.loader.exec_module(b); "
                        "r=subprocess.run(b.launcher_cmd(sys.argv[1:], 2, b._free_port()), cwd=b.ROOT); "
                        "raise SystemExit(r.returncode)"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2
