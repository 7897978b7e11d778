for v in default bigA bigB bigC; do
  if [ $v = default ]; then L=paper_2306_02687_b200/lib/libfe2rom_gpu.so; else L=paper_2306_02687_b200/lib/variants/lib_$v.so; fi
  FE2_LIB=$L timeout -s KILL 400 python tools/sweep.py --seconds 1 --which 3,4 --only n64_K400,n64_K4000,n128_K400,n128_K4000,config3 > gpurun_out/bigsweep_$v.jsonl 2>/dev/null
  echo "== $v"; python -c "
import json
for l in open('gpurun_out/bigsweep_$v.jsonl'):
    d=json.loads(l); print(f\"{d['cell']:22s} {d['evals_per_s']:.3e} evals/s  {d['frac_of_dmma_peak']:.2f} of DMMA\")"
done
