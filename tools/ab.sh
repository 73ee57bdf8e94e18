#!/bin/bash
# A/B on one box: tools/ab.sh <script> -- runs <script> with the current library
# and with paper_1709_07821_b200/libroaring_b200_old.so swapped in, twice each.
P=paper_1709_07821_b200
cp $P/libroaring_b200.so /tmp/new.so
for r in 1 2; do
  cp /tmp/new.so $P/libroaring_b200.so; echo "new:"; bash "$@"
  cp $P/libroaring_b200_old.so $P/libroaring_b200.so; echo "old:"; bash "$@"
done
cp /tmp/new.so $P/libroaring_b200.so
