# round 2: GPU suite incl. the fuzz cases, with the SweepArgs cleanup build
O=gpurun_out/r02ad
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py --steps 200 --warmup 20 --no-cpu-baseline > $O/bench_default.json 2> $O/bench_default.err
echo done
