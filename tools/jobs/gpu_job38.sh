#!/bin/bash
export PYTHONPATH=$PWD
GP_HOST_TIMING=1 timeout 600 python tools/e2e_probe.py 2>&1 | tail -30
