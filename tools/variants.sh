#!/bin/bash
# Build kernel-variant libraries for a sweep: tools/variants.sh NAME "DEFS" [NAME "DEFS" ...]
# -> paper_1412_0680_b200/_lib/v_NAME/libstmp_b200.so (select with STMP_LIB_PATH=...)
set -e
cd "$(dirname "$0")/.."
while [ $# -ge 2 ]; do
  STMP_BUILD_DIR=paper_1412_0680_b200/_lib/v_$1 STMP_NVCC_DEFS="$2" python -m paper_1412_0680_b200.build --force
  shift 2
done
