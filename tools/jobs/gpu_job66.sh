#!/bin/bash
export PYTHONPATH=$PWD
timeout 600 python tools/param_diff_probe.py 2>&1 | tail -17
