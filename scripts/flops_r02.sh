set -u
O=gpurun_out/${TAG:-r02e}; mkdir -p $O
M=gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma2_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd2_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul2_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-kernel-roofline --no-c3-anchor"
timeout 600 ncu --metrics $M -k regex:'k_phi_init|k_tag|k_kint|k_nb|k_count|k_scatter|k_gradient|k_probe|k_sweep' --clock-control none --csv --log-file $O/flops_c2.csv $B > $O/l2.log 2>&1
timeout 600 ncu --metrics $M -k regex:'k_phi_init|k_tag|k_kint|k_nb|k_count|k_scatter|k_gradient' --clock-control none --csv --log-file $O/flops_c3.csv $B --config C3 > $O/l3.log 2>&1
timeout 900 ncu --metrics $M -k regex:'k_phi_init|k_tag|k_kint|k_nb|k_count|k_scatter|k_gradient|k_probe' --clock-control none --csv --log-file $O/flops_c5.csv $B --config C5 > $O/l5.log 2>&1
