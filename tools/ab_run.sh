#!/bin/bash
# A/B kernel times of alternative libraries (run under gpurun): tools/ab_run.sh build/ab/libA.so build/ab/libB.so ...
for rep in 1 2; do
  for lib in "$@"; do
    DOCKSCREEN_LIB=$lib python bench.py --no-extras --no-cpu --no-e2e --steps 5 --warmup 2 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['kernel_ms'].items() if not isinstance(v,bool)})"
  done
done
