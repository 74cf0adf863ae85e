#!/bin/bash
# A/B of library variants on the C3 render: tools/ab_blend.sh lib1.so lib2.so ...
for lib in "$@"; do
  for rep in 1 2; do
    ODGS_B200_LIB=$lib python bench.py --no-train --no-large --no-cpu-baseline --steps 40 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value'],1), d['stages_ms'])"
  done
done
