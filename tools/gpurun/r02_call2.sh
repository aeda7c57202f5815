# round 2: GPU tests + first benches of the compact-ghost layout
mkdir -p gpurun_out/r02c
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 > gpurun_out/r02c/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r02c/pytest_gpu.log
for args in "--precision fp64" "--precision fp32" "--precision fp32 --workload patchy64" "--precision fp64 --layout aa" "--precision fp32 --layout aa"; do
  timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline $args >> gpurun_out/r02c/bench.jsonl 2>> gpurun_out/r02c/bench.err
done
echo done
