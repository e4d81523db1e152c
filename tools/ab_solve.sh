#!/bin/bash
# A/B of triangular-solve times across library builds in variants/ (development aid)
vs=$1; shift
for rep in 1 2; do
  for v in $vs; do
    if [ "$v" = cur ]; then lib=""; else lib=$PWD/variants/librq_$v.so; fi
    echo "== $v"; RQB_LIB=$lib python tools/solve_prof.py "$@"
  done
done
