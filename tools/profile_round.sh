set -x
python bench.py > gpurun_out/bench_r01c.log 2>&1; tail -1 gpurun_out/bench_r01c.log | head -c 600; echo
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01c.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-ns --no-advance --e2e-steps 3 > gpurun_out/ncu_l.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ns256_launches_r01c.csv python tools/ns_bench.py 256 1 > gpurun_out/ncu_ns.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:narrow3d_fast -s 3 -c 1 -o gpurun_out/prof_narrow_r01c python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-ns --no-advance --e2e-steps 3 > gpurun_out/ncu_n.log 2>&1
ncu --set full --import-source on --clock-control none -k "regex:ns_phase|prim_kernel|ns_assemble2|wdot_kernel|chem_kernel|ns_mixed" -c 12 -o gpurun_out/prof_ns_r01c python tools/ns_bench.py 128 1 > gpurun_out/ncu_ns2.log 2>&1
ls -la gpurun_out
