for cc in base none; do
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.max --clock-control $cc -k regex:gemm_tc --csv --log-file gpurun_out/r2z40_$cc.csv python tools/gemm_bench.py --reps 1 --burst 1 > gpurun_out/r2z40_$cc.log 2>&1
python - <<PY
import csv, io
lines = open('gpurun_out/r2z40_$cc.csv').read().splitlines()
st = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[st:]))))
cur = {}
for r in rows:
    cur.setdefault(r["ID"], {})[r["Metric Name"]] = r["Metric Value"]
for i, m in cur.items():
    print("$cc", i, "dram GB %.2f" % (float(m["dram__bytes_read.sum"].replace(",",""))/1e9), "clk %.0f MHz" % (float(m["sm__cycles_elapsed.avg.per_second"].replace(",",""))/1e6), "L2 hit", m["lts__t_sector_hit_rate.pct"], "ms %.3f" % (float(m["gpu__time_duration.sum"].replace(",",""))/1e6), "Mcyc %.2f" % (float(m["sm__cycles_elapsed.max"].replace(",",""))/1e6))
PY
done
