#!/bin/bash
# which engine feature the fused-step nondeterminism depends on (S = 2 in-process pipeline)
export PYTHONPATH=$PWD
C='{"data": "powerlaw", "kind": 2, "L": 8, "S": 2, "G": 1, "K": 8, "ep": 4}'
for extra in "GP_MERGED_G=0" "GP_BWD_CSR=0" "GP_LEAN=0" "GP_SPLIT=0 GP_TC_XFORM=0" "GP_PGRAD=simt"; do
timeout 300 python tools/det_probe.py "$C" 6 GP_FUSED_STEP=1 $extra
done
