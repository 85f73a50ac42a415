timeout 600 ncu --set full --import-source on -k regex:fft_ols -s 3 -c 1 -o gpurun_out/prof_fft_cfg4 python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_fft.log 2>&1
tail -2 gpurun_out/ncu_fft.log
