#!/bin/bash
# A/B of library variants on single C5 row bands: tools/ab_bands_stages.sh lib1.so lib2.so ...
for lib in "$@"; do
  ODGS_B200_LIB=$lib python tools/band_stages.py 2>&1 | tail -2 | sed "s|^|$lib |"
done
