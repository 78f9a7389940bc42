B200MOE_NCU_RANGE=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct --clock-control none --profile-from-start off -k regex:gemm_tc --csv --log-file gpurun_out/r2z38_step.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
python - <<'PY'
import csv, io
lines = open('gpurun_out/r2z38_step.csv').read().splitlines()
st = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[st:]))))
cur = {}
for r in rows:
    cur.setdefault(r["ID"], {})[r["Metric Name"]] = (r["Metric Value"], r["Metric Unit"])
for i, m in cur.items():
    print(i, {k: v for k, v in m.items()})
PY
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct --clock-control none -k regex:gemm_tc --csv --log-file gpurun_out/r2z38_alone.csv python tools/gemm_bench.py --routed --reps 1 --burst 1 > /dev/null 2>&1
python - <<'PY'
import csv, io
lines = open('gpurun_out/r2z38_alone.csv').read().splitlines()
st = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[st:]))))
cur = {}
for r in rows:
    cur.setdefault(r["ID"], {})[r["Metric Name"]] = (r["Metric Value"], r["Metric Unit"])
for i, m in list(cur.items())[:14]:
    print("alone", i, {k: v for k, v in m.items()})
PY
