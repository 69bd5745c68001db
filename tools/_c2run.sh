M=smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum
python tools/restore_iter1.py --c5
timeout 900 ncu --set full --metrics $M --clock-control none --import-source on -k regex:restore_sweep -c 1 -o gpurun_out/r02_restore_c5 python tools/restore_iter1.py --c5 > gpurun_out/ncu_rc5.log 2>&1
tail -1 gpurun_out/ncu_rc5.log
