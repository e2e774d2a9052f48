for v in 1 0 1 0; do echo "TP_TREE_LEVEL=$v"; TP_TREE_LEVEL=$v timeout 600 python scripts/bench_db.py --batches 16 | cut -c1-110; done
