for cap in 8192 4096 3000; do
  echo "== SFFT_FS_CAP=$cap"
  SFFT_FS_CAP=$cap python bench_configs.py --configs C4 --signals 256 --reps 4 --check 2 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d['config'], d['signals'], round(d['transforms_per_s'],1), 'ms', round(d['ms_per_batch'],3), 'gbs', round(d['bucketize_gbs']), d['support_identical'])
"
done
