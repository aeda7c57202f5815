# round 2: fp64 load-issue experiments (offset tables with selected addresses) and the
# cp.async sweep with fewer spills
O=gpurun_out/r02g
mkdir -p $O
S="--precision fp64;--precision fp32;--precision fp64 --layout aa"
bash tools/variant_bench.sh $O/v0.jsonl build/variants/desc.so build/variants/async2.so build/variants/off_select.so build/variants/desc.so -- "$S"
S1="--precision fp32;--precision fp32 --workload patchy64;--precision fp32 --layout aa"
LBM_SWEEP_VARIANT=1 bash tools/variant_bench.sh $O/v1.jsonl build/variants/desc.so build/variants/async2.so build/variants/off_select.so -- "$S1"
LBM_SWEEP_VARIANT=2 bash tools/variant_bench.sh $O/v2.jsonl build/variants/async2.so -- "--precision fp64;--precision fp32;--precision fp32 --workload patchy64"
echo done
