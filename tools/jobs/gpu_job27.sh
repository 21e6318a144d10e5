#!/bin/bash
# bisect: current tree (v0), HEAD libraries (v1), current engine + statically linked host C++ runtime (v2)
for v in v0 v1 v2; do
  if [ $v = v0 ]; then unset GP_LIBDIR; else export GP_LIBDIR=$PWD/variants/$v; fi
  timeout 150 python -m pytest tests/test_gpu_ipc.py -q -x -p no:cacheprovider -k same_process > gpurun_out/j27_$v.txt 2>&1; echo "$v ipc rc=$?"
  timeout 150 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "two_stages or three_stages" > gpurun_out/j27_${v}_par.txt 2>&1; echo "$v parity-s2 rc=$?"; tail -1 gpurun_out/j27_${v}_par.txt
done
