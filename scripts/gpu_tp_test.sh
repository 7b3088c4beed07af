# Exercise bench.py's multi-rank path (head shards, all-gather, max-over-ranks timing) with
# 2 ranks sharing the one GPU over gloo -- correctness of the plumbing, not a scaling number.
PA_BENCH_SAME_DEVICE=1 PA_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 20 --warmup 3 --config c2_alpaca ${TP_GATHER:+--tp-gather $TP_GATHER} \
  > gpurun_out/tp2_gloo.json 2> gpurun_out/tp2_gloo.err
echo rc=$?; cat gpurun_out/tp2_gloo.json; tail -5 gpurun_out/tp2_gloo.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29612 \
  bench.py --gpus 1 --steps 50 --warmup 3 > gpurun_out/tp1_torchrun.json 2> gpurun_out/tp1_torchrun.err
echo rc=$?; cut -c1-300 gpurun_out/tp1_torchrun.json; tail -3 gpurun_out/tp1_torchrun.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo rc=$?; cat gpurun_out/ref.json
