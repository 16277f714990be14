#!/bin/bash
# A/B alternative builds of liblongflow.so: tools/ab_libs.sh <workload> lib1.so lib2.so ...
w=$1; shift
for lib in "$@"; do
  cp $lib paper_2603_11504_b200/liblongflow.so
  echo "== $lib"; tools/sweep_split.sh $w 0
done
