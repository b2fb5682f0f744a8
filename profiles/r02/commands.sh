set -u
mkdir -p gpurun_out/r02
O=gpurun_out/r02
nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/alu_peaks.cu -o /tmp/alu_peaks && /tmp/alu_peaks > $O/alu_peaks.json 2>&1
M=gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-kernel-roofline --no-c3-anchor"
timeout 600 ncu --metrics $M -k regex:'k_phi_init|k_tag|k_kint|k_nb|k_count|k_scatter|k_gradient|k_probe|k_sweep' --clock-control none --csv --log-file $O/flops_c2.csv $B > $O/ncu_flops_c2.log 2>&1
timeout 600 ncu --metrics $M -k regex:'k_phi_init|k_tag|k_kint|k_nb|k_count|k_scatter|k_gradient' --clock-control none --csv --log-file $O/flops_c3.csv $B --config C3 > $O/ncu_flops_c3.log 2>&1
timeout 900 ncu --metrics $M -k regex:'k_phi_init|k_tag|k_kint|k_nb|k_count|k_scatter|k_gradient' --clock-control none --csv --log-file $O/flops_c5.csv $B --config C5 > $O/ncu_flops_c5.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $B > $O/ncu_launch.log 2>&1
timeout 600 python bench.py --slab --steps 3 --warmup 3 --no-e2e > $O/bench_slab1.json 2> $O/bench_slab1.err
timeout 600 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
