set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/m_smi.txt
timeout 400 python bench.py > gpurun_out/m_bench.log 2>&1
timeout 400 python bench.py --impl reference > gpurun_out/m_bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/m_launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/m_launch_run.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:el_decode_tc -s 1 -c 1 -o gpurun_out/m_decode320 python tools/profile_decode.py --B 320 --reps 2 > gpurun_out/m_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:splitk -s 2 -c 1 -o gpurun_out/m_splitk python tools/profile_step.py --B 32 --steps 1 > gpurun_out/m_ncu2.log 2>&1
timeout 300 python tools/time_stages.py --B 32 64 128 320 > gpurun_out/m_stages.log 2>&1
timeout 300 python tools/time_small_batch.py --B 16 32 64 128 > gpurun_out/m_small.log 2>&1
