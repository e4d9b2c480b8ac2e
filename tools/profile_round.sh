# The round's measurement commands (run under gpurun from the repo root; each
# ncu command only after the same command exited 0 without ncu).
set -x
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 600 gpurun_out/bench.json; echo
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1
# launch list + DRAM bytes of the NS RHS (full, advection-diffusion, chemistry)
python tools/ns_bench.py 256 1 > gpurun_out/nsb.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/ns256_launches.csv python tools/ns_bench.py 256 1 > gpurun_out/ncu_l.log 2>&1
# full sections of one NS RHS (its 6 kernels) and of the configs[1] kernel
ncu --set full --import-source on --clock-control none -k 'regex:ns_phase|prim_kernel|ns_assemble2' \
    -c 6 -o gpurun_out/prof_ns python tools/ns_bench.py 256 1 > gpurun_out/ncu_ns.log 2>&1
# executed FP64 operations per kernel (profiles/ncu_ns_fp64_ops_r02.json)
ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum \
    --clock-control none -k 'regex:ns_phase|prim_kernel|ns_assemble2' -c 6 --csv --log-file gpurun_out/ns_ops.csv \
    python tools/ns_bench.py 256 1 > gpurun_out/ncu_ops.log 2>&1
python tools/narrow_time.py 256 50 > gpurun_out/nt.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:narrow3d_fast -s 3 -c 1 \
    -o gpurun_out/prof_narrow python tools/narrow_time.py 256 50 > gpurun_out/ncu_n.log 2>&1
# one SDC and one MRSDC step at 128^3: shares and DRAM bytes per launch
python tools/advance_launches.py 128 mrsdc > gpurun_out/adv.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/adv_mrsdc.csv python tools/advance_launches.py 128 mrsdc > gpurun_out/ncu_a.log 2>&1
ls -la gpurun_out
