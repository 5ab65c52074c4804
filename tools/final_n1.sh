#!/bin/bash
# One-GPU validation + measurement pass (what the round-end driver runs, plus the ncu launch list):
# the GPU test suite, smoke(), bench.py (C2 + C3 / C5 sub-lines), --config 3, the reference arm.
# Outputs under gpurun_out/final/.
set -u
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > $O/tests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" >> $O/tests.log 2>&1
timeout 600 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err
timeout 400 python bench.py --config 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 400 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k[123]_|kp_" --csv \
  --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu.log 2>&1
echo done
