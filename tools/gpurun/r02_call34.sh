# round 2: final build on 2 GPUs -- multi-GPU tests, weak / strong bench lines, and the 1-GPU default line
O=gpurun_out/r02ag
mkdir -p $O
timeout 2400 python -m pytest tests/test_multi_gpu.py -m gpu -q --timeout 1200 > $O/pytest_multi_gpu_2.log 2>&1; echo "rc=$?" >> $O/pytest_multi_gpu_2.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > $O/bench_1gpu_default.json 2> $O/bench_1gpu_default.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29701 bench.py --gpus 2 > $O/bench_2gpu_default.json 2> $O/bench_2gpu_default.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29702 bench.py --gpus 2 --impl reference --steps 3 --warmup 1 > $O/bench_2gpu_reference.json 2> $O/bench_2gpu_reference.err
echo done
