# scratch driver (r02 session 7): ncu evidence for the GPT-2s reproducible launch (ring 6 x 4 splits, DSM reduce-scatter)
O=gpurun_out/r02s7; mkdir -p $O
timeout 600 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --csv --log-file $O/dram_gpt2s_fused.csv python tools/dram_bytes.py run gpt2s fused > $O/dram_gpt2s.log 2>&1; echo "dram rc=$?"
python tools/dram_bytes.py parse $O/dram_gpt2s_fused.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ff_chain_kernel -s 3 -c 1 -o $O/prof_gpt2s_dsmr \
  python tools/timeline.py gpt2s x3 cfg=6,4,128,128,3,4,1,1,16,16,96 > $O/ncu_gpt2s_full.log 2>&1; echo "ncu rc=$?"
ncu -i $O/prof_gpt2s_dsmr.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys,json
r=list(csv.reader(sys.stdin)); h=r[0]; u=r[1]; v=r[2]
want=['gpu__time_duration.sum','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active','dram__bytes_read.sum','dram__bytes_write.sum','lts__throughput.avg.pct_of_peak_sustained_elapsed','launch__grid_size','launch__cluster_dim_x','sm__cycles_elapsed.avg.per_second','l1tex__m_xbar2l1tex_read_bytes.sum']
print(json.dumps({w:(v[h.index(w)],u[h.index(w)]) for w in want if w in h}, indent=0))
" > $O/ncu_gpt2s_dsmr_summary.json; cat $O/ncu_gpt2s_dsmr_summary.json
