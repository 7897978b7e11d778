python paper_2306_02687_b200/build.py > /dev/null 2>&1 || echo BUILD_FAIL
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
timeout -s KILL 300 $CMD > gpurun_out/prof_plain.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_increment -s 19 -c 1 -o gpurun_out/prof_inc20 $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_increment -s 39 -c 1 -o gpurun_out/prof_inc40 $CMD > gpurun_out/ncu_full2.log 2>&1
echo "full2 rc=$?"
