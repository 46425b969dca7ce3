#!/bin/bash
# Evidence for profiles/: bench lines, launch lists, one ncu --set full step.
# Run on the GPU box:  bash tools/capture_round.sh <tag>
T=${1:-v9}
O=gpurun_out/$T
mkdir -p $O
python bench.py > $O/c2.json 2> $O/c2.err; echo "c2 rc=$?"
for w in c3_train_fp32_zipf c4_large_sharded_bf16 c5_latency_bf16 f4_tokens_bf16 f4_tokens_pertable_bf16; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-e2e > $O/$w.json 2> $O/$w.err; echo "$w rc=$?"
done
timeout 600 python bench.py --workload c4_large_sharded_bf16 --sharded --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/c4_sharded.json 2>/dev/null; echo "sharded rc=$?"
python bench.py --gate tanh --steps 20 --no-e2e --no-cpu-baseline > $O/c2_gate_tanh.json 2>/dev/null
python bench.py --update sgd --steps 20 --no-e2e --no-cpu-baseline > $O/c2_update_sgd.json 2>/dev/null
python bench.py --prologue --steps 20 --no-e2e --no-cpu-baseline > $O/c2_prologue.json 2>/dev/null
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/ref.json 2>/dev/null; echo "ref rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c2_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "launches rc=$?"
for w in c3_train_fp32_zipf c4_large_sharded_bf16; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --nvtx --nvtx-include "prof/" --csv --log-file $O/${w}_launches.csv python tools/prof_step.py $w > /dev/null 2>&1
  echo "$w launches rc=$?"
done
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "prof/" -o $O/c2_full \
    python tools/prof_step.py c2_mid_bf16 > $O/ncu_full.log 2>&1; echo "full rc=$?"
ncu -i $O/c2_full.ncu-rep --page raw --csv > $O/c2_full_raw.csv 2>/dev/null
