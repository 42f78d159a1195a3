out=gpurun_out/r02_s11_ep; mkdir -p $out
timeout 600 python -m pytest tests/test_layer_gpu.py -q -k "h_discard" > $out/pytest_discard.log 2>&1; echo "discard test rc=$?" >> $out/status.txt
for n in 4 8; do
  MOE_BENCH_ONE_GPU_TEST=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2954$n bench.py --gpus $n --steps 5 --warmup 3 > $out/ep$n.log 2>&1; echo "ep$n rc=$?" >> $out/status.txt
  MOE_BENCH_ONE_GPU_TEST=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n bench.py --gpus $n --steps 5 --warmup 3 --ep-transport nccl > $out/ep${n}_nccl.log 2>&1; echo "ep$n nccl rc=$?" >> $out/status.txt
done
MOE_BENCH_ONE_GPU_TEST=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29560 bench.py --gpus 2 --steps 5 --warmup 3 --scaling strong > $out/ep2_strong.log 2>&1; echo "ep2 strong rc=$?" >> $out/status.txt
tail -2 $out/pytest_discard.log >> $out/status.txt
cat $out/status.txt
for f in $out/ep*.log; do echo "== $f"; grep '^{' $f | head -1 | cut -c1-600; done
