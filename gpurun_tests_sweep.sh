export FE2_TRACE=${FE2_TRACE:-60}
python paper_2306_02687_b200/build.py > /dev/null 2>&1 || echo BUILD_FAIL
timeout -s KILL 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
unset FE2_TRACE
timeout -s KILL 1500 python tools/sweep.py --seconds 2 > gpurun_out/sweep_r01.jsonl 2> gpurun_out/sweep_r01.err; echo sweep rc=$?; tail -2 gpurun_out/sweep_r01.err
