#!/bin/bash
# C5 sweep time (tools/c5_cap.py) per library variant.  usage: c5_variants.sh base V ...
for v in "$@"; do
  if [ "$v" = "base" ]; then unset SW_LIB_VARIANT; else export SW_LIB_VARIANT=$v; fi
  echo "== $v"; python tools/c5_cap.py 4471054848 3221225472
done
