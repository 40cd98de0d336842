timeout 900 python -m pytest tests/test_gpu_sharding.py -q -p no:cacheprovider -x 2>&1 | tail -15
for cfg in headline 5 4; do
  timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -c 1500; echo
done
timeout 600 python bench.py --config 5 --scaling strong --steps 5 --warmup 3 2>&1 | tail -c 800; echo
TIDE_BENCH_ONE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -c 1500; echo
for cfg in 5 4; do
TIDE_BENCH_ONE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29556 bench.py --gpus 2 --config $cfg --steps 3 --warmup 3 2>&1 | tail -c 1200; echo
done
