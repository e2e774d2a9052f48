#!/bin/bash
# A/B of in-tree build variants (libtreepipe_b200.<name>.so) in one call: forward times, twice each.
for round in 1 2; do for v in "$@"; do echo "== $v (round $round)"; TP_LIB_VARIANT=$v bash scripts/fwd_times.sh; done; done
