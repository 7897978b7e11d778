V=paper_2306_02687_b200/lib/variants
echo "== cholu"; FE2_LIB=$V/lib_cholu.so python tools/cfg_run.py 24 400 65536 50 1 3 2>&1 | tail -3
echo "== cholu prof"; FE2_LIB=$V/lib_cholup.so python tools/cfg_run.py 24 400 65536 50 1 1 2>&1 | tail -2
echo "== base"; python tools/cfg_run.py 24 400 65536 50 1 3 2>&1 | tail -2
echo "== fs base"; python tools/cfg_run.py 32 600 32768 30 2 2 2>&1 | tail -2
for k in 10 12; do echo "== fs kw$k"; FE2_LIB=$V/lib_fskw$k.so python tools/cfg_run.py 32 600 32768 30 2 2 2>&1 | tail -1; done
