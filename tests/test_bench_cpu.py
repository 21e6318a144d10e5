"""bench.py contract checks that need no GPU: the reference arm (the reference's own trainer, whole
epochs) prints the same metric / config as the GPU arm, loads nothing from the product, and
--gpus must agree with WORLD_SIZE."""
import json
import os
import subprocess
import sys

import pytest

from oracle.blob import have_ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


@pytest.mark.skipif(not have_ref(), reason="oracle/_ref/ref_driver not built")
def test_reference_arm_line():
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    # run the arm in-process and report afterwards whether any product module or library got loaded
    probe = ("import runpy, sys\n"
             "sys.argv = ['bench.py', '--impl', 'reference', '--workload', 'er4k', '--steps', '2', '--warmup', '1']\n"
             "runpy.run_path('bench.py', run_name='__main__')\n"
             "maps = open('/proc/self/maps').read()\n"
             "print('PRODUCT_LOADED', any(m.startswith('paper_2308_10087_b200') for m in sys.modules), "
             "'libgpcuda' in maps or 'libgnnsim_b200' in maps)\n")
    r = subprocess.run([sys.executable, "-c", probe], cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    import bench
    assert line["impl"] == "reference" and line["metric"] == bench.METRIC and line["unit"] == "s/epoch"
    assert line["higher_is_better"] is False and line["steps"] == 2 and line["warmup"] == 1

    class A:
        workload, layers = "er4k", 0
    assert line["config"] == bench.workload_config(A, 1, 4)  # identical to the GPU arm's config
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] == 1 and cb["value"] == line["value"] > 0
    # er4k (8 layers) is measured whole, not projected
    assert cb["projection"] is False and set(cb["measured_epoch_s"]) == {"8"}
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    # the reference arm never imports the product package or maps its libraries
    assert "PRODUCT_LOADED False False" in r.stdout, r.stdout[-500:]


def test_gpus_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--impl", "reference"], cwd=ROOT,
                       capture_output=True, text=True, timeout=120, env=env)
    assert r.returncode != 0 and "disagrees with WORLD_SIZE" in (r.stderr + r.stdout)


def test_stage_ranges_match_the_product():
    import bench
    import paper_2308_10087_b200 as gp
    for L in (3, 8, 16, 64):
        for S in range(1, 9):
            if S <= L:
                assert bench.stage_ranges(L, S) == [tuple(x) for x in gp.make_stage_assignment(L, S)]
