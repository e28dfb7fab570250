#!/bin/bash
# One GPU-box pass that refreshes the judged evidence under gpurun_out/:
# bench lines (D default, E mixed + clay-only, batched B / C, D deterministic,
# reference arm), the launch list of the D bench and one `ncu --set full`
# capture of a fused k_particles launch at D and at E.
# Each ncu run follows the same command having exited 0 without ncu.
set -u
O=gpurun_out
python bench.py > $O/bench_D.json 2> $O/bench_D.err; echo "bench D rc=$?"
python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "bench ref rc=$?"
python bench.py --config E > $O/bench_E.json 2> $O/bench_E.err; echo "bench E rc=$?"
python bench.py --config E --clay-only --no-cpu-baseline > $O/bench_E_clay.json 2> $O/bench_E_clay.err; echo "bench E clay rc=$?"
python bench.py --config B --no-cpu-baseline > $O/bench_B.json 2> $O/bench_B.err; echo "bench B rc=$?"
python bench.py --config C --no-cpu-baseline > $O/bench_C.json 2> $O/bench_C.err; echo "bench C rc=$?"
python bench.py --deterministic --no-cpu-baseline > $O/bench_D_det.json 2> $O/bench_D_det.err; echo "bench D det rc=$?"
python bench.py --config A > $O/bench_A.json 2> $O/bench_A.err; echo "bench A rc=$?"
python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/bench_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_D.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launches.log 2>&1; echo "launch list rc=$?"
ncu --set full --import-source on --clock-control none -k regex:k_particles -s 41 -c 1 -f -o $O/kp_D \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_full.log 2>&1; echo "ncu full D rc=$?"
ncu --set full --import-source on --clock-control none -k regex:k_particles -s 41 -c 1 -f -o $O/kp_E \
    python bench.py --config E --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_full_E.log 2>&1; echo "ncu full E rc=$?"
python tools/bench_small.py > $O/small.json 2>&1; echo "small configs rc=$?"
python tools/bench_tasks.py --out $O/tasks.json > /dev/null 2>&1; echo "tasks rc=$?"
