#!/bin/bash
# A/B of library variants on one C4 view's backward: tools/ab_bwd.sh lib1.so lib2.so ...
for lib in "$@"; do
  echo "$lib $(ODGS_B200_LIB=$lib python tools/profile_c4_view.py 5 2>&1 | tail -1)"
done
