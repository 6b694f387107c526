# Final measurements of round 2c (run on the GPU box from the repo root); outputs -> gpurun_out/c_*
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/c_smi.txt
timeout 400 python bench.py > gpurun_out/c_bench.log 2>&1
timeout 400 python bench.py > gpurun_out/c_bench2.log 2>&1
timeout 400 python bench.py --impl reference > gpurun_out/c_bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/c_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/c_launch_run.log 2>&1
timeout 300 python tools/time_small_batch.py --B 8 16 32 64 128 > gpurun_out/c_small.log 2>&1
timeout 600 python tools/time_configs.py > gpurun_out/c_configs.log 2>&1
timeout 600 python tools/selfattn_bench.py > gpurun_out/c_selfattn.log 2>&1
timeout 300 python tools/mha_vs_el.py --B 32 320 > gpurun_out/c_mha.log 2>&1
timeout 300 python tools/time_fp32.py > gpurun_out/c_fp32.log 2>&1
timeout 300 python tools/step_timeline.py --B 32 320 --show 8 --json gpurun_out/c_timeline.jsonl > gpurun_out/c_timeline.txt 2>&1
