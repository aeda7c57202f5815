# round 2: 2 GPUs -- multi-GPU tests and weak-scaling bench lines with the round-2 kernels
O=gpurun_out/r02q
mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 2400 python -m pytest tests/test_multi_gpu.py -m gpu -q --timeout 1200 > $O/pytest_multi_gpu_2.log 2>&1; echo "rc=$?" >> $O/pytest_multi_gpu_2.log
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $1 bench.py --gpus 2 "${@:2}"; }
run 29511 --steps 200 --warmup 20 > $O/bench_2gpu_ldc256.json 2> $O/bench_2gpu_ldc256.err
run 29512 --steps 200 --warmup 20 --precision fp32 --workload patchy64 > $O/bench_2gpu_patchy64.json 2> $O/bench_2gpu_patchy64.err
run 29513 --steps 200 --warmup 20 --layout aa > $O/bench_2gpu_aa.json 2> $O/bench_2gpu_aa.err
run 29514 --steps 200 --warmup 20 --exchange nccl > $O/bench_2gpu_nccl.json 2> $O/bench_2gpu_nccl.err
run 29515 --steps 200 --warmup 20 --proc-grid 2,1,1 > $O/bench_2gpu_ldc256_x.json 2> $O/bench_2gpu_ldc256_x.err
run 29516 --steps 100 --warmup 10 --workload strong768 --no-e2e > $O/bench_2gpu_strong768.json 2> $O/bench_2gpu_strong768.err
echo done
