# round 2: AA kernels without wall logic (bounce-back list modes 1 / 2) + BB entries with inline
# masks: GPU suite, A/B, compute-sanitizer over tools/sanitize_cases.py
O=gpurun_out/r02l
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 400 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
S="--precision fp64;--precision fp32;--precision fp32 --workload patchy64;--precision fp64 --layout aa;--precision fp32 --layout aa"
bash tools/variant_bench.sh $O/ab.jsonl build/variants/bbl2.so build/variants/bbl.so -- "$S"
for tool in memcheck racecheck initcheck synccheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_cases.py > $O/sanitize_$tool.log 2>&1; echo "rc=$?" >> $O/sanitize_$tool.log
done
echo done
