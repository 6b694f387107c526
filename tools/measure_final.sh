set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/f_smi.txt
timeout 400 python bench.py > gpurun_out/f_bench.log 2>&1
timeout 400 python bench.py > gpurun_out/f_bench2.log 2>&1
timeout 400 python bench.py --impl reference > gpurun_out/f_bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/f_launch_run.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --graph-profiling node --csv --log-file gpurun_out/f_step32.csv python tools/profile_step.py --B 32 > gpurun_out/f_ps.log 2>&1
timeout 300 python tools/time_small_batch.py --B 16 32 64 128 > gpurun_out/f_small.log 2>&1
timeout 300 python tools/time_fp32.py > gpurun_out/f_fp32.log 2>&1
timeout 300 python tools/mha_vs_el.py --B 32 320 > gpurun_out/f_mha.log 2>&1
