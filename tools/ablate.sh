#!/bin/bash
# k_particles time per launch (config D, 256 envs) for the default build, the
# profiling-only ablations (abl_*: a stage removed, wrong physics) and the
# tuning variants (var_*). Build them first: make -C paper_2302_04659_b200 ablation
for v in base ${@:-abl_eigen abl_scatter abl_g2p var_cta4 var_cta6}; do
  if [ $v = base ]; then lib=paper_2302_04659_b200/libmsim_gpu.so; else lib=paper_2302_04659_b200/build/$v/libmsim_gpu.so; fi
  MSIM_GPU_LIB=$lib python bench.py --steps 2 --warmup 2 --envs 256 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', round(d['kernels']['k_particles']['avg_ms'],3), 'ms/launch', d['clocks']['sm_mhz'])"
done
