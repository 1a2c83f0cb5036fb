#!/bin/bash
# usage: bash tools/ab.sh out.jsonl libA.so libB.so ...   (interleaved rounds)
out=$1; shift
mkdir -p gpurun_out
for round in 1 2 3; do
  for lib in "$@"; do
    DKV_LIB=$lib timeout 600 python tools/ab.py >> gpurun_out/$out 2>> gpurun_out/ab.err
  done
done
