#!/bin/bash
# fused optimizer step nondeterminism: serialised launches, single stage
export PYTHONPATH=$PWD
C='{"data": "powerlaw", "kind": 2, "L": 8, "S": 2, "G": 1, "K": 8, "ep": 4}'
C1='{"data": "powerlaw", "kind": 2, "L": 8, "S": 1, "G": 1, "K": 8, "ep": 4}'
timeout 300 python tools/det_probe.py "$C" 6 GP_FUSED_STEP=1 CUDA_LAUNCH_BLOCKING=1
timeout 300 python tools/det_probe.py "$C1" 6 GP_FUSED_STEP=1
timeout 300 python tools/det_probe.py "$C" 6 GP_FUSED_STEP=1 GP_TC_XFORM=0
timeout 300 python tools/det_probe.py "$C" 6
