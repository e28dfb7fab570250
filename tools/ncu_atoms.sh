for v in base var_nocellsort; do
  if [ $v = base ]; then lib=paper_2302_04659_b200/libmsim_gpu.so; else lib=paper_2302_04659_b200/build/$v/libmsim_gpu.so; fi
  MSIM_GPU_LIB=$lib ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__inst_executed.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum --clock-control none -k regex:k_particles -s 41 -c 1 --csv python bench.py --steps 1 --warmup 1 --envs 1024 --no-cpu-baseline > gpurun_out/ncu_atoms_$v.csv 2>/dev/null
done
