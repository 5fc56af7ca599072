#!/bin/bash
# compute-sanitizer tier (run on the GPU box): memcheck, racecheck, synccheck
# over tools/sanitize_workload.py, plus the column-blocked K1 schedule and the
# graph-replayed loops in their own processes.  Logs -> gpurun_out/sanitize/.
out=gpurun_out/sanitize
mkdir -p $out
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # name tool env...
  local name=$1 tool=$2; shift 2
  env "$@" timeout 1500 $CS --tool $tool --error-exitcode 9 --print-limit 50 \
      python tools/sanitize_workload.py > $out/$name.log 2>&1
  echo "$name rc=$? $(grep -c '^ok' $out/$name.log) steps; $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $out/$name.log | tail -1)"
}
run memcheck memcheck
run racecheck racecheck
run synccheck synccheck
run memcheck_colblock memcheck KZ_K1_SLICE_MB=0.1 KZ_K1_MINDEG=16 KZ_SANITIZE_PART=cg
run racecheck_colblock racecheck KZ_K1_SLICE_MB=0.1 KZ_K1_MINDEG=16 KZ_SANITIZE_PART=cg
run memcheck_graphs memcheck KZ_GRAPHS=1 KZ_SANITIZE_PART=lrc
run racecheck_graphs racecheck KZ_GRAPHS=1 KZ_SANITIZE_PART=cg
