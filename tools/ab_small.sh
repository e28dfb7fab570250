#!/bin/bash
# ms per env step of the single-scene configs (tools/bench_small.py) for the
# in-tree library and variant builds, two alternating passes
for pass in 1 2; do
for v in base "$@"; do
  if [ $v = base ]; then lib=paper_2302_04659_b200/libmsim_gpu.so; else lib=paper_2302_04659_b200/build/$v/libmsim_gpu.so; fi
  echo "$v $(MSIM_GPU_LIB=$lib python tools/bench_small.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: round(v['ms_per_env_step'], 3) for k, v in d.items()})")"
done; done
