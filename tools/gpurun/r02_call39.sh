# round 2: 96 fuzz cases + the full GPU suite of the final build
O=gpurun_out/r02al
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
echo done
