nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_event_reasons.active,temperature.gpu --format=csv -lms 100 > gpurun_out/clk.csv &
SMI=$!
timeout 300 python tools/time_loop.py --sched 0 --n 100,1000,1000,100,10
timeout 300 python tools/time_loop.py --sched 1 --n 100,1000,1000,100,10
kill $SMI
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/clk.csv')))[1:]
import collections
print(len(rows))
for r in rows[::10]: print(",".join(x.strip() for x in r))
PY
