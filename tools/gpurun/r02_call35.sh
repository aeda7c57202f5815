# round 2: the driver's launch lines with the final bench.py (stdout = one JSON line)
O=gpurun_out/r02ah
mkdir -p $O
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29711 bench.py --gpus 2 --steps 200 --warmup 20 > $O/bench_2gpu.stdout 2> $O/bench_2gpu.stderr
timeout 600 python bench.py --steps 200 --warmup 20 > $O/bench_1gpu.stdout 2> $O/bench_1gpu.stderr
wc -l $O/*.stdout > $O/lines.txt
echo done
