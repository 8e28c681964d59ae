# scratch driver (r02 session 7): final checks at HEAD -- GPU suite, smoke, smoke under ncu (as the driver runs it)
O=gpurun_out/r02s7; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests_final.log 2>&1; echo "pytest rc=$?"; tail -1 $O/gpu_tests_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_final.log 2>&1; echo "smoke rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ncu_smoke_final.csv \
  python -c "import __graft_entry__ as g; g.smoke()" > $O/ncu_smoke_final.log 2>&1; echo "ncu smoke rc=$?"
grep -c ff_chain $O/ncu_smoke_final.csv; grep "ff_chain" $O/ncu_smoke_final.csv | awk -F'","' '{print $5, $NF}' | cut -c1-120
