#!/bin/bash
# Full-forward times (scripts/ablate_fwd.py): lone n=1 and n=44 stages (16 layers), the 7-stage group (4 layers).
for n in 1 44 45,35,29,23,17,11,3; do timeout 300 python scripts/ablate_fwd.py --n $n --masks "" --iters 40 2>&1 | grep "full forward"; done
