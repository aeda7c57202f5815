# round 2: fuzz cases with random exchange modes
O=gpurun_out/r02ai
mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_fuzz.py -m gpu -q --timeout 900 > $O/pytest_fuzz.log 2>&1; echo "rc=$?" >> $O/pytest_fuzz.log
echo done
