# round 2: programmatic dependent launch of the bounce-back list (pdl) vs the final build
O=gpurun_out/r02aj
mkdir -p $O
cp build/variants/pdl.so paper_1007_1388_b200/liblbm_b200.so
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_aa.py tests/test_gpu_fuzz.py tests/test_gpu_fullsize.py -m gpu -q --timeout 900 > $O/pytest_pdl.log 2>&1; echo "rc=$?" >> $O/pytest_pdl.log
cp build/variants/final.so paper_1007_1388_b200/liblbm_b200.so
S="--precision fp64;--precision fp32;--precision fp64 --layout aa;--precision fp32 --layout aa;--precision fp32 --workload patchy64"
bash tools/variant_bench.sh $O/ab.jsonl build/variants/pdl.so build/variants/final.so build/variants/pdl.so build/variants/final.so -- "$S"
echo done
