O=gpurun_out/e2e1; mkdir -p $O
run() { env "$@" timeout 120 python scripts/e2e_sweep.py >> $O/sweep.jsonl 2>> $O/err.log; }
run X=1
run SG_PROBE_DOWN1=1
run SG_PROBE_RING=8
run SG_PROBE_RING=2
run SG_PROBE_CHUNK=262144
run SG_PROBE_CHUNK=1048576
run SG_PROBE_CHUNK=2097152
run SG_PROBE_CHUNK=4194304 SG_PROBE_RING=3
run SG_PROBE_CHUNK=131072 SG_PROBE_RING=8
run SG_PROBE_CHUNK=1048576 SG_PROBE_RING=8
run SG_PROBE_CHUNK=1048576 SG_PROBE_DOWN1=1
python scripts/pcie_bw.py > $O/pcie.json 2>&1
