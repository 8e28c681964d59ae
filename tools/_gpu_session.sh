# scratch driver (r02 session 6q): OPT M=32768 DRAM bytes / time with streaming A / E evict_first
set -x
O=gpurun_out/r02s6q; mkdir -p $O
for v in 0x0 0x1000 0x1400; do
  timeout 600 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file $O/dram_$v.csv python tools/dram_bytes.py run opt13b_m32768 fused variant=$v > /dev/null 2>&1
  python tools/dram_bytes.py parse $O/dram_$v.csv > $O/dram_$v.json; echo $v; cat $O/dram_$v.json
done
timeout 900 python tools/ab_variant.py 0x0 0x1400 opt13b_m32768 gpt67b steps=30 > $O/ab.log 2>&1; grep variant $O/ab.log
