#!/bin/bash
# per-kernel durations of the config-5 setup + one cycle (ncu launch list, summed by kernel name)
python tools/run_cycles.py config5 1 > gpurun_out/plain.log 2>&1; echo "plain rc=$?"; cat gpurun_out/plain.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/setup_launches.csv python tools/run_cycles.py config5 1 > gpurun_out/ncu_setup.log 2>&1; echo "ncu rc=$?"
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open('gpurun_out/setup_launches.csv')) if len(r) > 10]
h = rows[0]; ki = h.index('Kernel Name'); mi = h.index('Metric Name'); vi = h.index('Metric Value'); ui = h.index('Metric Unit')
t = collections.defaultdict(float); n = collections.Counter(); b = collections.defaultdict(float)
for r in rows[1:]:
    name = r[ki].split('(')[0][:60]
    v = float(r[vi].replace(',', ''))
    if r[mi] == 'gpu__time_duration.sum':
        u = r[ui]; v = v * {'ns': 1e-6, 'us': 1e-3, 'ms': 1.0, 'msecond': 1.0, 'usecond': 1e-3, 'nsecond': 1e-6, 'second': 1e3}.get(u, 1e-6)
        t[name] += v; n[name] += 1
    else:
        u = r[ui]; b[name] += v * {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'Tbyte': 1e12}.get(u, 1)
for k, v in sorted(t.items(), key=lambda kv: -kv[1])[:25]:
    print(f"{v:10.2f} ms  {n[k]:5d} launches  {b[k]/1e9:9.2f} GB  {k}")
print("total", round(sum(t.values()), 1), "ms")
PY
