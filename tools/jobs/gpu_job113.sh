#!/bin/bash
# determinism of the config the fused-step probe flagged, under several engine settings
export PYTHONPATH=$PWD
C='{"data": "powerlaw", "kind": 2, "L": 8, "S": 2, "G": 1, "K": 8, "ep": 4}'
H='{"data": "powerlaw", "kind": 2, "L": 8, "S": 2, "G": 2, "K": 8, "ep": 8, "cs": 3, "ps": 1}'
timeout 300 python tools/det_probe.py "$C" 6
timeout 300 python tools/det_probe.py "$C" 6 GP_FUSED_STEP=0
timeout 300 python tools/det_probe.py "$C" 6 GP_REMASK_OVERLAP=0
timeout 300 python tools/det_probe.py "$C" 6 GP_WAVE=1
timeout 300 python tools/det_probe.py "$H" 4
timeout 300 python tools/det_probe.py "$H" 4 GP_FUSED_STEP=0
