set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_csr_tma -s 40 -c 30 -o /tmp/prof_l1 python tools/profile_step.py --config 3 --maxit 4 > gpurun_out/ncu_l1.log 2>&1
ncu -i /tmp/prof_l1.ncu-rep --page raw --csv > gpurun_out/ncu_l1_raw.csv 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/ncu_l1_raw.csv')))
h=rows[0]
for i,r in enumerate(rows[2:]):
    print(i, r[h.index('Kernel Name')][:40], r[h.index('gpu__time_duration.sum')])
PY
for k in 0 1 2 3 4 5 6 7 8 9 10 11 12 13 14 15; do
  ncu -i /tmp/prof_l1.ncu-rep --page source --csv --print-source sass --launch-skip $k --launch-count 1 > gpurun_out/ncu_l1_sass_$k.csv 2>&1
done
ls -la gpurun_out | head -40
