#!/bin/bash
# two-sweep reinit: bitwise tests, oracle reinit tests, A/B bench (C2, C3, C5)
set -u
O=gpurun_out/${TAG:-ts}; mkdir -p $O
python -m paper_2512_11473_b200.build > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_tsweep_gpu.py -q -x -rf > $O/pytest_ts.log 2>&1; echo "rc=$?" >> $O/pytest_ts.log
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_window_gpu.py -q -rf -k "reinit or drift or c3 or c5 or smoke" > $O/pytest_parity.log 2>&1; echo "rc=$?" >> $O/pytest_parity.log
for cfg in C2 C3 C5; do
  st=10; [[ $cfg == C5 ]] && st=3
  timeout 600 python bench.py --config $cfg --steps $st --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_$cfg.json 2> $O/bench_$cfg.err
  SG_TSWEEP=0 timeout 600 python bench.py --config $cfg --steps $st --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_${cfg}_single.json 2> $O/bench_${cfg}_single.err
done
