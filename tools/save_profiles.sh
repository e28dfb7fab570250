#!/bin/bash
# Copy the evidence of tools/profile_round.sh from gpurun_out/ into profiles/ under a tag:
#   bash tools/save_profiles.sh r02a
set -e
T=$1
O=gpurun_out
SHA=$(git rev-parse --short HEAD)
for f in D E E_clay B C D_det A; do [ -f $O/bench_$f.json ] && tail -1 $O/bench_$f.json > profiles/${T}_bench_$f.json; done
tail -1 $O/bench_ref.json > profiles/${T}_bench_reference.json
[ -f $O/small.json ] && cp $O/small.json profiles/${T}_small_configs.json
[ -f $O/tasks.json ] && cp $O/tasks.json profiles/${T}_tasks_D.json
{ echo "# ncu launch list ($T, git $SHA): \`python bench.py --steps 1 --warmup 1 --no-cpu-baseline\` (config D, 1024 envs, B200), whole process incl. setup"
  echo "# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: compare SHARES)"
  python3 tools/launch_summary.py $O/launches_D.csv; } > profiles/${T}_launches_D.txt
SUB=paper_2302_04659_b200/csrc/msim_substep.cu
L() { grep -n "$1" $SUB | head -1 | cut -d: -f1; }
a=$(L "^__device__ __forceinline__ void item_rounds"); b=$(L "// ---------------- G2P of this cycle")
c=$(L "// ---------------- binning of the (new) position"); d=$(L "// ---------------- write back in bucket order")
e=$(L "// ---------------- per-thread scatter"); f=$(L "// ---------------- flush the round"); g=$(L "^__device__ __forceinline__ void particles_cta")
for C in D E; do
  [ -f $O/kp_$C.ncu-rep ] || continue
  { echo "# ncu --set full --clock-control none --import-source on -k regex:k_particles -s 41 -c 1 python bench.py --config $C --steps 1 --warmup 1 --no-cpu-baseline  (B200, git $SHA)"
    echo "# regions by msim_substep.cu line ranges of this build (fix_rn = helpers; 'other' = CUDA headers: atomics, shuffles)"
    NCU_LAUNCH=0 python3 profiles/ncu_summary.py $O/kp_$C.ncu-rep 30 msim_device.cuh:1-900=constitutive_sdf msim_common.cuh:1-2000=common \
      msim_substep.cu:1-$((a-1))=helpers msim_substep.cu:$a-$((b-1))=pp_load msim_substep.cu:$b-$((c-1))=g2p_returnmap \
      msim_substep.cu:$c-$((d-1))=bin_penalty_payload msim_substep.cu:$d-$((e-1))=writeback_keys msim_substep.cu:$e-$((f-1))=scatter \
      msim_substep.cu:$f-$((g-1))=flush msim_substep.cu:$g-$((g+160))=item_setup; } > profiles/${T}_ncu_k_particles_$C.txt
done
python3 - "$T" "$SHA" <<'PY'
import json, os, re, sys
tag, sha = sys.argv[1], sys.argv[2]
out = {}
for cfg, n in (("D", 1024 * 16384), ("E", 4000000)):
    p = f"profiles/{tag}_ncu_k_particles_{cfg}.txt"
    if not os.path.exists(p):
        continue
    t = open(p).read()
    def val(name):
        m = re.search(name + r" ([\d.]+) (G|M)byte", t)
        return float(m.group(1)) * (1e9 if m.group(2) == "G" else 1e6)
    r, w = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    out[cfg] = {"dram_bytes_per_particle_per_fused_launch": (r + w) / n, "git_sha": sha, "capture": p,
                "particles": n}
    print(cfg, "traffic B/particle per fused launch", (r + w) / n)
old = json.load(open("profiles/traffic.json")) if os.path.exists("profiles/traffic.json") else {}
old = {k: v for k, v in old.items() if k in ("D", "E")}
old.update(out)
json.dump(old, open("profiles/traffic.json", "w"), indent=1)
PY
