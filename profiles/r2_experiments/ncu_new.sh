summ() {
python - "$1" <<'PY'
import csv, sys
rows=list(csv.reader(open(sys.argv[1])))
h=rows[0]; i_n=h.index("Metric Name"); i_v=h.index("Metric Value"); i_u=h.index("Metric Unit"); i_s=h.index("Section Name"); i_k=h.index("Kernel Name")
keep=["Duration","DRAM Throughput","L1/TEX Cache Throughput","L2 Cache Throughput","Compute (SM) Throughput","Registers Per Thread","Achieved Occupancy","Theoretical Occupancy","Executed Ipc Active","Issue Slots Busy","No Eligible","L1/TEX Hit Rate","L2 Hit Rate","Dynamic Shared Memory Per Block","Warp Cycles Per Issued Instruction","Mem Busy","Max Bandwidth","Bank conflicts","Grid Size","Block Size"]
print(rows[1][i_k][:100])
for r in rows[1:]:
    if any(k.lower() == r[i_n].lower() for k in keep): print("  ", r[i_s][:30].ljust(30), r[i_n][:44].ljust(44), r[i_v], r[i_u])
PY
}
for k in k_fs_cols k_fs_rows k_vote_sliced k_fold_rows; do
  ncu --set full --clock-control none -k regex:$k -s 1 -c 1 -o gpurun_out/n_$k -f python bench_configs.py --configs C5a --signals 128 --reps 1 --check 0 > gpurun_out/n_$k.log 2>&1
  ncu -i gpurun_out/n_$k.ncu-rep --page details --csv > gpurun_out/n_$k.csv
  ncu -i gpurun_out/n_$k.ncu-rep --page raw --csv | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2] if len(r)>2 else r[1]
for name in ['dram__bytes_read.sum','dram__bytes_write.sum','gpu__time_duration.sum','lts__t_sectors_srcunit_tex_op_read.sum','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','smsp__inst_executed.sum']:
    if name in h: print('   raw', name, v[h.index(name)])
"
  summ gpurun_out/n_$k.csv
done
for k in k_cols k_pe_peel; do
  ncu --set full --clock-control none -k regex:$k -s 2 -c 1 -o gpurun_out/n_$k -f python bench_configs.py --configs C4 --signals 128 --reps 1 --check 0 > gpurun_out/n_$k.log 2>&1
  ncu -i gpurun_out/n_$k.ncu-rep --page details --csv > gpurun_out/n_$k.csv
  summ gpurun_out/n_$k.csv
done
