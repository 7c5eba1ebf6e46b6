# Launch list (per-kernel device time) of one full C4 left move (ISO solver included).
mkdir -p gpurun_out
timeout 300 python tools/prof_move.py c4 full > gpurun_out/prof_full.out 2>&1 && \
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_full_move.csv python tools/prof_move.py c4 full > gpurun_out/ncu_full.log 2>&1
echo "rc=$?" > gpurun_out/rc_prof.txt
