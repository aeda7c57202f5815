# round 2: AA PULL skips the dead ghost scatter of uniform-wall x sides (aaw3) + setup kernel per (patch, side)
O=gpurun_out/r02aa
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
S="--precision fp64 --layout aa;--precision fp32 --layout aa;--precision fp64;--precision fp32"
bash tools/variant_bench.sh $O/ab.jsonl build/variants/aaw3.so build/variants/aaw2.so build/variants/aaw3.so -- "$S"
echo done
