#!/bin/bash
# compute-sanitizer pass over every kernel family at small shapes
# (tools/sanitize_cases.py) plus the 2-rank peer-memory exchange from the pure
# C++ host (build/bin/ep_p2p_demo: two processes sharing the GPU through CUDA
# IPC).  One log per (tool, case) under gpurun_out/<tag>/; summary.txt holds
# the ERROR SUMMARY line of each.
tag=${1:-sanitize}
out=gpurun_out/$tag
mkdir -p $out
CS=/usr/local/cuda/bin/compute-sanitizer
CASES=${CASES:-cfg1 lm mt256 onesm split static graph route cache host ep1}
TOOLS=${TOOLS:-memcheck racecheck synccheck}
: > $out/summary.txt
for tool in $TOOLS; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check full"
  [ $tool = racecheck ] && extra="--racecheck-report all"
  for c in $CASES; do
    timeout ${CASE_TIMEOUT:-900} $CS --tool $tool $extra --error-exitcode 9 \
      python tools/sanitize_cases.py $c > $out/${tool}_$c.log 2>&1
    rc=$?
    echo "$tool $c rc=$rc $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' $out/${tool}_$c.log | tail -1)" >> $out/summary.txt
  done
  timeout ${CASE_TIMEOUT:-900} $CS --tool $tool $extra --target-processes all --error-exitcode 9 \
    build/bin/ep_p2p_demo --world 2 --devices 1 --tokens 512 --experts 16 --hidden-dim 1024 --steps 2 \
    --dir /tmp/ep_san_$tool > $out/${tool}_ep2.log 2>&1
  rc=$?
  echo "$tool ep2 rc=$rc $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' $out/${tool}_ep2.log | tail -1)" >> $out/summary.txt
done
python tools/sanitize_summary.py $out > $out/classified.txt
cat $out/summary.txt $out/classified.txt
