export FE2_TRACE=${FE2_TRACE:-60}
python paper_2306_02687_b200/build.py > /dev/null 2>&1 || echo BUILD_FAIL
timeout -s KILL 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -25
