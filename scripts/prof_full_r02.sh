set -u
O=gpurun_out/r02f; mkdir -p $O
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-kernel-roofline --no-c3-anchor"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_probe|k_kint' -s 2 -c 2 -o $O/prof_probe_kint $B > $O/ncu_pk.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_sweep' -s 25 -c 1 -o $O/prof_sweep $B > $O/ncu_sw.log 2>&1
ls -la $O
