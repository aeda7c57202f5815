# round 2: 4 GPUs, final build (after the one-cell-thick fix and the JSON-only stdout)
O=gpurun_out/r02ak
mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 3000 python -m pytest tests/test_multi_gpu.py -m gpu -q --timeout 1500 > $O/pytest_multi_gpu_4.log 2>&1; echo "rc=$?" >> $O/pytest_multi_gpu_4.log
run() { n=$1; port=$2; shift 2; if [ $n = 1 ]; then timeout 900 python bench.py "$@"; else timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $port bench.py --gpus $n "$@"; fi; }
p=29600
for n in 1 2 4; do
  p=$((p+1)); run $n $p --steps 500 --warmup 20 > $O/bench_${n}gpu_ldc256.json 2> $O/bench_${n}gpu_ldc256.err
  p=$((p+1)); run $n $p --steps 200 --warmup 20 --precision fp32 --workload patchy64 > $O/bench_${n}gpu_patchy64.json 2> $O/bench_${n}gpu_patchy64.err
  p=$((p+1)); run $n $p --steps 200 --warmup 20 --workload weak384 --no-e2e > $O/bench_${n}gpu_weak384.json 2> $O/bench_${n}gpu_weak384.err
  p=$((p+1)); run $n $p --steps 50 --warmup 5 --workload strong768 --no-e2e > $O/bench_${n}gpu_strong768.json 2> $O/bench_${n}gpu_strong768.err
  p=$((p+1)); run $n $p --steps 200 --warmup 20 --layout aa > $O/bench_${n}gpu_aa.json 2> $O/bench_${n}gpu_aa.err
done
p=$((p+1)); run 4 $p --steps 200 --warmup 20 --proc-grid 2,2,1 > $O/bench_4gpu_ldc256_221.json 2> $O/bench_4gpu_ldc256_221.err
p=$((p+1)); run 4 $p --steps 200 --warmup 20 --exchange nccl > $O/bench_4gpu_nccl.json 2> $O/bench_4gpu_nccl.err
echo done
