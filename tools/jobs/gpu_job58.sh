#!/bin/bash
for u in 1 2 5; do echo "== unroll $u"; ./tools/fwd_bench_u$u 2>&1 | grep -E "tile<4,100>|tile<1,4,100>|differing"; done
