B=paper_2105_04779_b200/csrc/build_base/libbase.so
N=paper_2105_04779_b200/libelattn_gpu.so
python -m pytest tests -m gpu -x -q -k "qexp or fused or small or step" 2>&1 | tail -2
for lib in $B $N $B $N; do echo "== $lib"; python tools/time_small_batch.py --B 4 8 16 --lib $lib; done
python tools/step_timeline.py --B 8 --show 6 | tail -8
