"""Reader for the ``GPBLOB01`` files written by oracle/ref_driver.cpp (test infrastructure)."""
import os
import subprocess
import numpy as np

_DT = {1: np.uint8, 2: np.uint32, 3: np.uint64, 4: np.float32, 5: np.float64, 6: np.int64}
HERE = os.path.dirname(os.path.abspath(__file__))
REF_DRIVER = os.path.join(HERE, "_ref", "ref_driver")


def read_blob(path):
    out = {}
    with open(path, "rb") as f:
        data = f.read()
    if data[:8] != b"GPBLOB01":
        raise ValueError(f"{path}: not a blob file")
    at = 8
    while at < len(data):
        n = int.from_bytes(data[at:at + 4], "little"); at += 4
        name = data[at:at + n].decode(); at += n
        dt, nd = data[at], data[at + 1]; at += 2
        dims = [int.from_bytes(data[at + 8 * i:at + 8 * i + 8], "little") for i in range(nd)]; at += 8 * nd
        dtype = np.dtype(_DT[dt])
        cnt = int(np.prod(dims)) if dims else 1
        arr = np.frombuffer(data, dtype=dtype, count=cnt, offset=at).reshape(dims).copy()
        at += cnt * dtype.itemsize
        out[name] = arr
    return out


def have_ref():
    return os.path.exists(REF_DRIVER)


def run_ref(cmd, out_path, timeout=600, **kw):
    """Run the reference driver and return its blob as a dict of arrays."""
    args = [REF_DRIVER, cmd] + [f"{k}={v}" for k, v in kw.items()] + [f"out={out_path}"]
    r = subprocess.run(args, capture_output=True, text=True, timeout=timeout)
    if r.returncode != 0:
        raise RuntimeError(f"ref_driver {cmd} failed ({r.returncode}): {r.stderr.strip()}")
    return read_blob(out_path)
