#!/bin/bash
# A/B of library builds on one box: tools/ab_libs.sh <script> [args...] runs the
# script with tools/ab_libs/new.so and tools/ab_libs/old.so swapped in, twice
# each, alternating (build them here: make; cp the .so; git stash; make; cp).
P=paper_1709_07821_b200
cp $P/libroaring_b200.so /tmp/cur.so
for r in 1 2; do
  for v in new old; do
    cp tools/ab_libs/$v.so $P/libroaring_b200.so
    echo -n "$v: "; python "$@"
  done
done
cp /tmp/cur.so $P/libroaring_b200.so
