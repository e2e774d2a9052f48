#!/bin/bash
# Build an in-tree library variant for same-box A/B runs (loaded with TP_LIB_VARIANT=<name>):
#   bash scripts/build_variant.sh <name> "<extra nvcc flags>"
# then rebuild the default library (objects are cached by mtime, so sources are touched).
set -e
name=$1; extra=$2
cd "$(dirname "$0")/.."
L=paper_2504_04104_b200
touch $L/csrc/*.cu
TP_NVCC_EXTRA="$extra" python -m paper_2504_04104_b200.build > /dev/null
cp $L/libtreepipe_b200.so $L/libtreepipe_b200.$name.so
touch $L/csrc/*.cu
python -m paper_2504_04104_b200.build > /dev/null
echo "built $L/libtreepipe_b200.$name.so ($extra)"
