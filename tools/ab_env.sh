#!/bin/bash
# usage: bash tools/ab_env.sh out.jsonl "label:VAR=val VAR2=val" ...   (interleaved rounds, one lib)
out=$1; shift
mkdir -p gpurun_out
for round in 1 2 3; do
  for spec in "$@"; do
    label=${spec%%:*}; envs=${spec#*:}
    env $envs AB_LABEL=$label timeout 600 python tools/ab.py >> gpurun_out/$out 2>> gpurun_out/ab.err
  done
done
