# round 2: AA kernels store the uniform-wall sides' bounce-back too (aaw) vs sw
O=gpurun_out/r02x
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
S="--precision fp64 --layout aa;--precision fp32 --layout aa;--precision fp64;--precision fp32"
bash tools/variant_bench.sh $O/ab.jsonl build/variants/aaw.so build/variants/sw.so build/variants/aaw.so -- "$S"
echo done
