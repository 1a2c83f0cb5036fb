# pair vs single backward at other BASELINE shapes (one group each): C5 (32/4 heads, P=16K), C2
mkdir -p gpurun_out
for shape in 32,16384,2048,32,4 16,4096,1024,32,8; do
  for r in 1 2; do
    AB_SHAPE=$shape AB_LABEL=single_$shape AB_REP=0 AB_REPS=3 timeout 300 python tools/ab.py >> gpurun_out/shapes_ab.jsonl 2>>gpurun_out/pair_ab.err
    DKV_BWD_PAIR=1 AB_SHAPE=$shape AB_LABEL=pair_$shape AB_REP=0 AB_REPS=3 timeout 300 python tools/ab.py >> gpurun_out/shapes_ab.jsonl 2>>gpurun_out/pair_ab.err
  done
done
