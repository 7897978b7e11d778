for v in w8s3 w16s6 w12s4; do
  FE2_LIB=paper_2306_02687_b200/lib/variants/lib_$v.so timeout -s KILL 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/sweep_$v.json 2> gpurun_out/sweep_$v.err
  echo "$v rc=$? $(python -c "import json;d=json.load(open('gpurun_out/sweep_$v.json'));print(round(d['value']/1e6,3),'M evals/s', round(d['roofline']['executed_dmma_tflops'],2))")"
done
