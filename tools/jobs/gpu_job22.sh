#!/bin/bash
echo split; timeout 600 python tools/e2e_probe2.py 2>&1 | tail -16
echo fused; GP_SPLIT=0 timeout 600 python tools/e2e_probe2.py 2>&1 | tail -8
