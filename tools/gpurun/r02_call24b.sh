# round 2: AA side-wall stores + phantom partners re-reading their own cell (aaw2) vs sw
O=gpurun_out/r02x2
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
S="--precision fp64 --layout aa;--precision fp32 --layout aa;--precision fp64;--precision fp32;--precision fp32 --workload patchy64"
bash tools/variant_bench.sh $O/ab.jsonl build/variants/aaw2.so build/variants/sw.so build/variants/aaw2.so -- "$S"
echo done
