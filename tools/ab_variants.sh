#!/bin/bash
# tools/ab_variants.sh "<lib names in tools/ab_libs, no .so>" <script> [args...]:
# runs the script once per library build per round (two rounds, interleaved).
P=paper_1709_07821_b200
cp $P/libroaring_b200.so /tmp/cur.so
for r in 1 2; do
  for v in $1; do
    cp tools/ab_libs/$v.so $P/libroaring_b200.so
    echo -n "$v: "; python "${@:2}"
  done
done
cp /tmp/cur.so $P/libroaring_b200.so
