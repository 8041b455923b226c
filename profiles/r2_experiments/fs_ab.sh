python -m pytest tests/test_gpu_c5grid.py tests/test_gpu_bucketize.py tests/test_gpu_runners.py -x -q -m gpu 2>&1 | tail -4
for v in 0 1; do
  echo "== SFFT_NO_FS_POW2=$v"
  if [ $v = 1 ]; then export SFFT_NO_FS_POW2=1; fi
  python bench_configs.py --configs C4,C5a,C5b --signals 256 --reps 3 --check 2 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d['config'], d['signals'], round(d['transforms_per_s'],1), 'ms', round(d['ms_per_batch'],3), 'frac', round(d['frac_of_measured_hbm'],4), d['support_identical'], d['max_rel_coeff_err'])
"
done
