# scratch driver (r02 session 6p): DRAM bytes at OPT M=32768, fused vs cuBLAS
set -x
O=gpurun_out/r02s6p; mkdir -p $O
for imp in fused cublas_eager cublas_fused_epilogue; do
  timeout 600 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file $O/dram_opt32k_$imp.csv python tools/dram_bytes.py run opt13b_m32768 $imp > /dev/null 2>&1
  python tools/dram_bytes.py parse $O/dram_opt32k_$imp.csv > $O/dram_opt32k_$imp.json; echo $imp; cat $O/dram_opt32k_$imp.json
done
