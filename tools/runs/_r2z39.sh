for cc in base none base none; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct --clock-control $cc -k regex:gemm_tc -c 2 --csv --log-file gpurun_out/r2z39.csv python tools/gemm_bench.py --only "dgrad1 store" --reps 1 --burst 1 > /dev/null 2>&1
python - <<PY
import csv, io
lines = open('gpurun_out/r2z39.csv').read().splitlines()
st = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[st:]))))
cur = {}
for r in rows:
    cur.setdefault(r["ID"], {})[r["Metric Name"]] = r["Metric Value"]
for i, m in cur.items():
    print("$cc", i, "dram GB %.2f" % (float(m["dram__bytes_read.sum"].replace(",",""))/1e9), "clk %.0f MHz" % (float(m["sm__cycles_elapsed.avg.per_second"].replace(",",""))/1e6), "L2 hit", m["lts__t_sector_hit_rate.pct"], "ms %.3f" % (float(m["gpu__time_duration.sum"].replace(",",""))/1e6))
PY
done
