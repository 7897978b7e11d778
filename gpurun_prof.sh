python paper_2306_02687_b200/build.py > /dev/null 2>&1 || echo BUILD_FAIL
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launches rc=$?"
$CMD > gpurun_out/prof_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:newton_round -s 40 -c 2 -o gpurun_out/prof_round $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
$CMD > gpurun_out/prof_plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_commit -s 20 -c 1 -o gpurun_out/prof_commit $CMD > gpurun_out/ncu_commit.log 2>&1
echo "commit rc=$?"
ls -la gpurun_out
