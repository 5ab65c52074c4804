# Final-tree runs behind profiles/bench_{n2,n4,c3n4,c4n4,c5n4}_r01.json (a 4-GPU gpurun box):
#   gpurun --gpus 4 -- 'bash tools/scale_r01.sh'
mkdir -p gpurun_out/scale
run() {  # run <n> <log> <bench args...>
  n=$1; log=$2; shift 2
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n "$@" > gpurun_out/scale/$log.log 2>&1
  echo $log $?; tail -1 gpurun_out/scale/$log.log | cut -c1-200
}
for n in 2 4; do run $n c2n$n; done
run 4 c3n4 --config 3 --steps 50
run 4 c5n4 --config 5
run 4 c4n4 --config 4
