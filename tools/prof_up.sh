# ncu --set full of the finest-level prolongation under a TMG_UPT variant: bash tools/prof_up.sh 3
python -m paper_1903_10367_b200.build > /dev/null 2>&1
export TMG_UPT=$1
CMD="python tools/run_cycles.py config5 3"
$CMD > gpurun_out/plain.log 2>&1; echo "plain rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k3_up_tile -s 3 -c 1 -o gpurun_out/prof_upt$1 $CMD > gpurun_out/ncu_upt.log 2>&1; echo "ncu rc=$?"
