#!/bin/bash
# Round-2 capture: smoke, GPU tests, bench lines (C2 headline, C3, C5 with probe,
# reference arm), ncu launch lists (C2, C5) and executed-arithmetic counts.
set -u
O=gpurun_out/${TAG:-r02b}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 900 python bench.py --config C5 --steps 5 --warmup 2 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-kernel-roofline --no-c3-anchor"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $B > $O/ncu_launch.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv $B --config C5 > $O/ncu_launch_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_probe|k_sweep' -s 20 -c 2 -o $O/prof_c2 $B > $O/ncu_c2.log 2>&1
ls -la $O > $O/ls.txt
