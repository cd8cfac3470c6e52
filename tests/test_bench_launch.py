"""bench.py's contract plumbing on CPU: `--gpus N` without torchrun spawns N
ranks itself (the driver's launch shape; here over gloo with --dry-run), and
the reference arm / cpu_baseline leg never import the product package (they
time the reference's own code from oracle/_ref, so libpact_cuda.so must not
be loaded in that process)."""
import ast
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gpus_n_spawns_n_ranks():
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    assert lines[0]["n_gpus"] == 2 and lines[0]["requested"] == 2


def _imports(fn: ast.FunctionDef):
    mods = set()
    for node in ast.walk(fn):
        if isinstance(node, ast.Import):
            mods.update(a.name for a in node.names)
        elif isinstance(node, ast.ImportFrom) and node.module:
            mods.add(node.module)
    return mods


def test_reference_arm_does_not_import_the_product():
    tree = ast.parse(open(os.path.join(ROOT, "bench.py")).read())
    fns = {n.name: n for n in tree.body if isinstance(n, ast.FunctionDef)}
    for name in ("run_reference", "cpu_baseline_leg", "ref_frame_signals"):
        mods = _imports(fns[name])
        assert not any(m.startswith("paper_2409_10876_b200") for m in mods), (name, mods)
    wd = ast.parse(open(os.path.join(ROOT, "workload_defs.py")).read())
    mods = _imports(wd)
    assert not any(m.startswith("paper_2409_10876_b200") for m in mods), mods
