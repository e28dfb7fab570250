#!/bin/bash
# Time share of k_particles stages: same bench with profiling-only builds.
for v in base eigen scatter g2p prefetch; do
  if [ $v = base ]; then lib=paper_2302_04659_b200/libmsim_gpu.so; else lib=paper_2302_04659_b200/build/abl_$v/libmsim_gpu.so; fi
  MSIM_GPU_LIB=$lib python bench.py --steps 2 --warmup 2 --envs 256 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', round(d['kernels']['k_particles']['avg_ms'],3), 'ms/launch', d['clocks'])"
done
