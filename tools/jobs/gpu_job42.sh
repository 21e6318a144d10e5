#!/bin/bash
for b in "" _minb5 _minb6; do echo "== fwd_bench$b"; ./tools/fwd_bench$b 2>&1 | grep -E "split gather k_fwd8<GCN2,2,1>|split k_bwd8<AGG,LAYER,2,1>|differing"; done
