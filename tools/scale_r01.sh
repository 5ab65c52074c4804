mkdir -p gpurun_out/scale
for n in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2960$n bench.py --gpus $n > gpurun_out/scale/c2n$n.log 2>&1; echo C2N$n $?; tail -1 gpurun_out/scale/c2n$n.log | cut -c1-200
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29614 bench.py --gpus 4 --config 3 --steps 50 > gpurun_out/scale/c3n4.log 2>&1; echo C3N4 $?; tail -1 gpurun_out/scale/c3n4.log | cut -c1-200
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29615 bench.py --gpus 4 --config 5 > gpurun_out/scale/c5n4.log 2>&1; echo C5N4 $?; tail -1 gpurun_out/scale/c5n4.log | cut -c1-200
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29616 bench.py --gpus 4 --config 4 > gpurun_out/scale/c4n4.log 2>&1; echo C4N4 $?; tail -1 gpurun_out/scale/c4n4.log | cut -c1-200
