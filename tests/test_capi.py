"""The drop-in boundary: the in-tree C-ABI libraries load and export every symbol that
include/gnnpipe.h declares; the GPU engine refuses to run without a device (no CPU
fallback). No compute calls here."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gnnpipe.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b((?:gp|gs)_[a-z0-9_]+)\s*\(", src)))


def exported(path):
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if line.strip()}


def test_header_declares_both_layers():
    names = declared()
    assert "gp_create" in names and "gp_run_epoch" in names and "gp_link_nccl" in names
    assert "gs_train_pipeline" in names and "gs_make_chunks" in names
    assert len(names) > 40


def test_every_declared_symbol_is_exported(gp):
    host, dev = gp.lib_paths()
    have = exported(host) | exported(dev)
    missing = [n for n in declared() if n not in have]
    assert not missing, missing
    gp_syms = [n for n in declared() if n.startswith("gp_")]
    assert all(n in exported(dev) for n in gp_syms), "device entry points must live in libgpcuda.so"


def test_libraries_are_sm100a_only():
    dev = os.path.join(ROOT, "paper_2308_10087_b200", "lib", "libgpcuda.so")
    out = subprocess.run(["cuobjdump", "--list-elf", dev], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_abi_version_and_loud_failure_without_device(gp):
    lib = gp._L()
    assert lib.gp_abi_version() == 1
    if gp.device_count() > 0:
        pytest.skip("a CUDA device is visible")
    specs = gp.build_layer_specs(gp.ModelConfig(kind=0, layers=2, hidden=8), 4, 2)
    with pytest.raises(gp.GpuEngineError):
        gp.StageEngine(num_vertices=10, num_chunks=1, specs=specs, stage=0, num_stages=1, layer_range=(0, 2),
                       hidden=8, num_classes=2, dropout=0.5, seed=1)
    ds = gp.Dataset.synthetic_er(50, 0.1, 1, 4, 2, 1)
    import numpy as np
    with pytest.raises(gp.GpuEngineError):
        gp.train_pipeline(ds, np.zeros(50, np.uint32), 1, gp.TrainOptions(model=gp.ModelConfig(kind=0, layers=2)))


def test_sass_contains_256bit_gathers():
    """The hot SpMM uses sm_100 256-bit vector loads with the L2 evict-last hint."""
    dev = os.path.join(ROOT, "paper_2308_10087_b200", "lib", "libgpcuda.so")
    sass = subprocess.run(["cuobjdump", "-sass", dev], capture_output=True, text=True).stdout
    assert "LDG.E.NA.ELL2.256" in sass


def test_libraries_do_not_interpose_torch():
    """Loading the engine before torch must not break torch (RTLD_LOCAL load)."""
    import subprocess
    import sys
    code = ("import paper_2308_10087_b200 as gp; gp.device_count(); import torch.distributed as d; "
            "import torch.fx; print('ok')")
    r = subprocess.run([sys.executable, "-c", code], cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]


def test_sass_contains_tcgen05_and_async_copies():
    """The parameter-gradient GEMM issues tcgen05 MMAs (UTC*MMA) reading TMEM back (LDTM); the tiled
    transforms stage rows with cp.async (LDGSTS)."""
    dev = os.path.join(ROOT, "paper_2308_10087_b200", "lib", "libgpcuda.so")
    sass = subprocess.run(["cuobjdump", "-sass", dev], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass or "UTCMMA" in sass
    assert "LDTM" in sass
    assert "LDGSTS" in sass
