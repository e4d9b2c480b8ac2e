B="python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-advance --ns-steps 1 --e2e-steps 3"
for i in 1 2; do
SMC_LIB_PATH=$PWD/build_ab/libsmc_old.so $B > gpurun_out/ab_old$i.json 2>gpurun_out/ab_old$i.err
$B > gpurun_out/ab_new$i.json 2>gpurun_out/ab_new$i.err
done

