#!/bin/bash
./tools/fwd_bench 2>&1 | grep -E "tile<1,4,100>|without"
