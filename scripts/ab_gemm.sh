#!/bin/bash
# A/B of in-tree build variants on K2 alone (scripts/gemm_knobs.py, fix-up mode 0) and on forwards.
for v in "$@"; do echo "== $v"; TP_LIB_VARIANT=$v timeout 300 python scripts/gemm_knobs.py --shape gu,qkv,o,down --n 1,16,48 --fixup 0 --stages 8; done
bash scripts/ab_variants.sh "$@"
