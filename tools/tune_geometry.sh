#!/bin/bash
# usage: tools/tune_geometry.sh "<geometries>" "<query numbers>"
for g in $1; do
  for q in $2; do
    echo -n "tile=$g q=$q: "
    SWB200_TILE=$g python tools/profile_scan.py $q 3 | tail -1
  done
done
