set -x
python -m paper_1903_10367_b200.build > /dev/null 2>&1 || true
CMD="python tools/run_cycles.py config5 3"
$CMD > gpurun_out/plain.log 2>&1; echo "plain rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k3_up_cell -s 3 -c 1 -o gpurun_out/prof_up $CMD > gpurun_out/ncu_up.log 2>&1; echo "up rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k3_top2 -s 1 -c 1 -o gpurun_out/prof_top2 $CMD > gpurun_out/ncu_top2.log 2>&1; echo "top rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k3_smooth2r -s 1 -c 1 -o gpurun_out/prof_sm2 $CMD > gpurun_out/ncu_sm2.log 2>&1; echo "sm rc=$?"
