mkdir -p gpurun_out/r02a
nvidia-smi > gpurun_out/r02a/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02a/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r02a/pytest_gpu.log
export LBM_SWEEP_IMPL=tma
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r02a/tma_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_tma -s 5 -c 2 -o gpurun_out/r02a/tma_full python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r02a/tma_ncu.log 2>&1
echo done
