set -x
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/gputest_full.log
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k_|^void k_' -c 4000 --csv --log-file gpurun_out/launches_raw.csv python bench.py --steps 1 --warmup 1 --batch 2048 --slots 2048 --no-e2e --no-cpu > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_group_fold -c 1 -o gpurun_out/gf_full -f python bench.py --steps 1 --warmup 0 --batch 512 --slots 512 --no-e2e --no-cpu > gpurun_out/ncu_gf_full.log 2>&1
ncu -i gpurun_out/gf_full.ncu-rep --page details --csv > gpurun_out/gf_full_details.csv
ncu -i gpurun_out/gf_full.ncu-rep --page raw --csv > gpurun_out/gf_full_raw.csv
tail -3 gpurun_out/gputest_full.log; tail -c 300 gpurun_out/bench_c3.err; head -c 400 gpurun_out/bench_c3.json
