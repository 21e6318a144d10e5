#!/bin/bash
# after ordering every upload before the engine's streams (settle_uploads) and the stream-ordered
# step-table upload: determinism of the configurations the fused step had exposed
export PYTHONPATH=$PWD
C='{"data": "powerlaw", "kind": 2, "L": 8, "S": 2, "G": 1, "K": 8, "ep": 4}'
H='{"data": "powerlaw", "kind": 2, "L": 8, "S": 2, "G": 2, "K": 8, "ep": 8, "cs": 3, "ps": 1}'
timeout 300 python tools/det_probe.py "$C" 8 GP_FUSED_STEP=1
timeout 300 python tools/det_probe.py "$H" 6 GP_FUSED_STEP=1
timeout 300 python tools/det_probe.py "$C" 6
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider > gpurun_out/j116_tests.txt 2>&1; echo "parity rc=$?"; tail -1 gpurun_out/j116_tests.txt
GP_FUSED_STEP=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider > gpurun_out/j116_tests_fused.txt 2>&1; echo "parity fused rc=$?"; tail -1 gpurun_out/j116_tests_fused.txt
