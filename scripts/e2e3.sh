O=gpurun_out/e2e3; mkdir -p $O
for c in 1945444 1966080 1572864 2097152 1048576 1900000; do SG_PROBE_CHUNK=$c timeout 120 python scripts/e2e_sweep.py >> $O/sweep.jsonl 2>> $O/err.log; done
