#!/bin/bash
# Build libslq_b200.so variants with extra nvcc defines into variants/<name>/ (experiments only):
#   tools/build_variants.sh name1="-DSLQ_SPMM_MINB4=4" name2="..."
# then run with SLQ_LIB_PATH=variants/<name>/libslq_b200.so.  Restores the default build afterwards.
set -e
cd "$(dirname "$0")/.."
for spec in "$@"; do
  name="${spec%%=*}"; defs="${spec#*=}"
  mkdir -p variants/$name
  SLQ_NVCC_FLAGS="$defs" python -c "from paper_2003_01282_b200 import build; build.build(force=True)"
  cp paper_2003_01282_b200/libslq_b200.so variants/$name/
done
python -c "from paper_2003_01282_b200 import build; build.build(force=True)"
