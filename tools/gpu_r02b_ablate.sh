# bottleneck ablations of the 128-query backward (profile build; wrong results by design)
for ab in 0 1 2 3; do
  A2D_ABLATE=$ab timeout 300 python tools/bwd_prof.py > gpurun_out/r3_ablate_$ab.json 2>&1
  echo "ablate=$ab $(python -c "import json; d=json.load(open('gpurun_out/r3_ablate_$ab.json')); print(round(d['bwd_tflops'],1), d['mma'])")"
done
