#!/bin/bash
# Round-2 multi-GPU runs on one box (N = number of visible GPUs): the default decode line (C2), C3
# prefill, and BASELINE configs 4 / 5 as written (8 nodes) with 8 / N domains per GPU, plus the
# multi-GPU oracle check. Outputs under gpurun_out/scale/.
set -u
N=$(python -c "import torch; print(torch.cuda.device_count())")
mkdir -p gpurun_out/scale
run() {   # name, args...
  local name=$1; shift
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 500)) "$@" > gpurun_out/scale/$name.json 2> gpurun_out/scale/$name.err
  echo "$name rc=$?"; tail -c 300 gpurun_out/scale/$name.json; echo
}
run xcheck_n$N tools/exchange_check.py
run c2_n$N bench.py --gpus $N
run c3_n$N bench.py --gpus $N --config 3 --steps 30
K=$((8 / N))
if [ $K -ge 1 ]; then
  run c4_8dom_n$N bench.py --gpus $N --config 4 --domains-per-gpu $K --steps 20
  run c5_8dom_n$N bench.py --gpus $N --config 5 --domains-per-gpu $K --steps 20
fi
