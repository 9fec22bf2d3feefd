# Paper Table III-style tile-width sweep on the paper's tensors A and B
# (PAPER.md:412-433), R = 32, through the reference-schema harness
mkdir -p gpurun_out
timeout 900 python -m paper_2510_14891_b200 sweep --shape 401,201,12,501 --ranks 32 --variants tile,b200 \
  --tile-widths 2,4,6,8,12 --reps 3 --out gpurun_out/table3_A.csv > gpurun_out/table3_A.log 2>&1
timeout 900 python -m paper_2510_14891_b200 sweep --shape 129,129,129,12,39 --ranks 32 --variants tile,b200 \
  --tile-widths 2,4,6,8,12 --reps 3 --out gpurun_out/table3_B.csv > gpurun_out/table3_B.log 2>&1
cat gpurun_out/table3_A.agg.csv gpurun_out/table3_B.agg.csv; tail -2 gpurun_out/table3_A.log
