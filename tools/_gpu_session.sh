# scratch driver (r02 session 7): the N-rank bench path (2 ranks sharing the one GPU) at HEAD
O=gpurun_out/r02s7; mkdir -p $O
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 \
  bench.py --gpus 2 --steps 50 --warmup 3 --no-extra --no-cpu > $O/bench_n2.json 2> $O/bench_n2.err; echo "rc=$?"
tail -c 600 $O/bench_n2.json; tail -3 $O/bench_n2.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 \
  bench.py --impl reference --gpus 2 --steps 2 --warmup 3 > $O/bench_n2_ref.json 2> $O/bench_n2_ref.err; echo "ref rc=$?"
tail -c 300 $O/bench_n2_ref.json
