#!/bin/bash
# A/B of factor times across library builds in variants/ (development aid):
#   tools/ab_factor.sh "v1 v2 ..." cfg...   (v = variants/librq_<v>.so; "cur" = in-tree build)
vs=$1; shift
for rep in 1 2; do
  for v in $vs; do
    if [ "$v" = cur ]; then lib=""; else lib=$PWD/variants/librq_$v.so; fi
    echo "== $v"; RQB_LIB=$lib python tools/factor_prof.py "$@"
  done
done
