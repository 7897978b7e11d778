python paper_2306_02687_b200/build.py > /dev/null 2>&1 || echo BUILD_FAIL
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:newton_round -s 40 -c 2 -o gpurun_out/prof_round2 $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
