#!/bin/bash
# Evidence for profiles/ (round 2): bench lines, launch lists, ncu --set full
# of the C4 sharded step (the headline) and of C2.  Run on the GPU box:
#   bash tools/capture_round.sh <tag>
T=${1:-r02}
O=gpurun_out/$T
mkdir -p $O
timeout 900 python bench.py > $O/c4.json 2> $O/c4.err; echo "c4 (default) rc=$?"
for w in c2_mid_bf16 c3_train_fp32_zipf c5_latency_bf16 f4_tokens_bf16 f4_tokens_pertable_bf16; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-e2e > $O/$w.json 2> $O/$w.err; echo "$w rc=$?"
done
timeout 600 python bench.py --unsharded --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/c4_unsharded.json 2>/dev/null; echo "unsharded rc=$?"
timeout 600 python bench.py --transport nccl --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/c4_nccl.json 2>/dev/null; echo "nccl rc=$?"
python bench.py --workload c2_mid_bf16 --gate tanh --steps 20 --no-e2e --no-cpu-baseline > $O/c2_gate_tanh.json 2>/dev/null
python bench.py --workload c2_mid_bf16 --update sgd --steps 20 --no-e2e --no-cpu-baseline > $O/c2_update_sgd.json 2>/dev/null
python bench.py --workload c2_mid_bf16 --prologue --steps 20 --no-e2e --no-cpu-baseline > $O/c2_prologue.json 2>/dev/null
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/ref.json 2>/dev/null; echo "ref rc=$?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --nvtx --nvtx-include "prof/" --csv --log-file $O/c4_launches.csv python tools/prof_sharded.py > /dev/null 2>&1
echo "c4 launches rc=$?"
for w in c2_mid_bf16 c3_train_fp32_zipf c5_latency_bf16; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --nvtx --nvtx-include "prof/" --csv --log-file $O/${w}_launches.csv python tools/prof_step.py $w > /dev/null 2>&1
  echo "$w launches rc=$?"
done
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "prof/" -o $O/c4_full \
    python tools/prof_sharded.py > $O/ncu_full.log 2>&1; echo "c4 full rc=$?"
ncu -i $O/c4_full.ncu-rep --page raw --csv > $O/c4_full_raw.csv 2>/dev/null
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "prof/" -o $O/c2_full \
    python tools/prof_step.py c2_mid_bf16 > $O/ncu_full_c2.log 2>&1; echo "c2 full rc=$?"
ncu -i $O/c2_full.ncu-rep --page raw --csv > $O/c2_full_raw.csv 2>/dev/null
# the roofline kernels' DRAM traffic -> profiles/traffic.json (run here; copy back)
python tools/traffic_json.py $T c4_large_sharded_bf16_xchg=$O/c4_full_raw.csv c2_mid_bf16=$O/c2_full_raw.csv > $O/traffic.log 2>&1
cp profiles/traffic.json $O/traffic.json
rm -f $O/*.ncu-rep
# the scorer's phase timelines (MSN_SELECT_TS build)
if [ -f paper_2602_07526_b200/libmsn_pkm_ts.so ]; then
  for c in c4_large_sharded_bf16 c2_mid_bf16 c5_latency_bf16 c3_train_fp32_zipf; do
    MSN_LIB=paper_2602_07526_b200/libmsn_pkm_ts.so timeout 200 python tools/select_ts.py $c >> $O/select_ts.txt 2>&1
  done
fi
# C5 warm phase times (20 calls per graph) and the column-segment A/B
for m in 1 2 4; do MSN_SELECT_SPLIT=$m timeout 120 python tools/c5_phases.py >> $O/c5_phases.txt 2>&1; done
timeout 120 python tools/c5_phases.py >> $O/c5_phases.txt 2>&1
