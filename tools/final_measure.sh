set -x
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest.log
python bench.py > gpurun_out/bench_final.log 2>&1
python bench.py --trimul > gpurun_out/bench_trimul_final.log 2>&1
python tools/step_profile.py 4 gpurun_out/step_profile_4blk.txt > gpurun_out/step_profile.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6100 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_ -o gpurun_out/r02b_attn_tri python tools/prof_attn.py tri 1 > gpurun_out/ncu_attn.log 2>&1
ls -la gpurun_out
