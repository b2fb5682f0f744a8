O=gpurun_out/e2e2; mkdir -p $O
timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 4 > $O/bench_default.json 2> $O/err1.log
SG_PROBE_CHUNK=2097152 timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 4 > $O/bench_2m.json 2> $O/err2.log
timeout 120 python scripts/e2e_sweep.py >> $O/sweep.jsonl 2>> $O/err.log
SG_PROBE_CHUNK=2097152 timeout 120 python scripts/e2e_sweep.py >> $O/sweep.jsonl 2>> $O/err.log
python scripts/pcie_bw.py > $O/pcie.json 2>&1
