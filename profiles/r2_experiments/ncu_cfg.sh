# usage: ncu_cfg.sh CONFIG SIGNALS
python bench_configs.py --configs $1 --signals $2 --reps 2 --check 0 2>&1 | cut -c1-300 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k_|^void k_' -c 3000 --csv --log-file gpurun_out/$1.csv python bench_configs.py --configs $1 --signals $2 --reps 1 --check 0 > gpurun_out/$1.log 2>&1
python - <<PY
import csv, collections
rows=[r for r in csv.reader(open("gpurun_out/$1.csv")) if len(r)>10]
h=rows[0]; ik=h.index("Kernel Name"); iv=h.index("Metric Value")
agg=collections.OrderedDict()
for r in rows[1:]:
    k=r[ik].split('(')[0]; e=agg.setdefault(k,[0.0,0]); e[0]+=float(r[iv].replace(',',''))/1e6; e[1]+=1
tot=sum(e[0] for e in agg.values())
print("total", tot)
for k,e in sorted(agg.items(), key=lambda x:-x[1][0])[:14]: print(f"{e[0]:9.3f} ms {100*e[0]/tot:5.1f}% n={e[1]:3d} {k}")
PY
