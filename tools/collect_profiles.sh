#!/bin/bash
# Copy the judged artefacts of the last tools/gpu_full.sh run from gpurun_out/ (scratch) into
# profiles/ (tracked), named per round:  bash tools/collect_profiles.sh r02
R=${1:-r02}
P=profiles
G=gpurun_out
first_json() { python - "$1" "$2" <<'PY'
import json, sys
for line in open(sys.argv[1]):
    if line.startswith("{"):
        json.dump(json.loads(line), open(sys.argv[2], "w"), indent=1)
        break
PY
}
first_json $G/bench_default.json $P/${R}_bench_config5.json
first_json $G/bench_ref.json $P/${R}_bench_reference_config5.json
first_json $G/bench_shard1.json $P/${R}_bench_config5_sharded_1rank.json
for w in config1 config2 config3 config4; do first_json $G/bench_$w.json $P/${R}_bench_$w.json; done
cp $G/launches_config5.csv $P/${R}_config5_launches_dram.csv
cp $G/traffic.json $P/traffic.json
cp $G/smoke.log $P/${R}_smoke.txt
tail -3 $G/pytest_gpu.log > $P/${R}_pytest_gpu.txt
for k in k3_top4r k3_smc k3_up_dict k3_rap_y k3_rap_out; do
  if [ -f $G/prof_$k.ncu-rep ]; then
    { echo "ncu --set full --clock-control none, one launch of $k, config 5 (python tools/run_cycles.py config5 3)";
      python tools/ncu_brief.py $G/prof_$k.ncu-rep; echo; echo "hottest source lines (instructions / stall samples):";
      python tools/ncu_lines.py $G/prof_$k.ncu-rep 25; } > $P/${R}_ncu_$k.txt 2>&1
  fi
done
# SASS instruction census of the default config-5 kernels (TMA, bulk copies, fp64 FMA)
{ echo "cuobjdump -sass paper_1903_10367_b200/libtmg.so: instruction counts per kernel";
  cuobjdump -sass paper_1903_10367_b200/libtmg.so | python tools/sass_census.py; } > $P/${R}_sass_census.txt
ls $P | grep $R
