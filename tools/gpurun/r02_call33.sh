# round 2: 48 fuzz cases + the final build's bench lines of the four 256^3 configurations
O=gpurun_out/r02af
mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py -m gpu -q --timeout 900 > $O/pytest_fuzz_parity.log 2>&1; echo "rc=$?" >> $O/pytest_fuzz_parity.log
S="--precision fp64;--precision fp32;--precision fp64 --layout aa;--precision fp32 --layout aa;--precision fp32 --workload patchy64"
bash tools/variant_bench.sh $O/ab.jsonl build/variants/final.so build/variants/final.so -- "$S"
echo done
