#!/bin/bash
export PYTHONPATH=$PWD
timeout 900 python tools/fused_probe.py 2>&1 | tail -8
