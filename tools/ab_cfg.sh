#!/bin/bash
# usage: ab_cfg.sh "<bench.py args>" variant...  -- k_particles ms/launch and value for the in-tree library
# and variant builds, two alternating passes (same box)
args=$1; shift
for pass in 1 2; do
for v in base "$@"; do
  if [ $v = base ]; then lib=paper_2302_04659_b200/libmsim_gpu.so; else lib=paper_2302_04659_b200/build/$v/libmsim_gpu.so; fi
  MSIM_GPU_LIB=$lib python bench.py $args --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', '$args', round(d['kernels']['k_particles']['avg_ms'],4), 'ms/launch', round(d['value']/1e9,3), 'G', d['clocks']['sm_mhz'])"
done; done
