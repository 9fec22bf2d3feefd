mkdir -p gpurun_out
for shape in "128 128 128 128" "128 16384 128" "16384 128 128" "128 128 16384" "256 256 256 16"; do
  timeout 300 python tools/sweep.py --shape $shape --ranks 256 --rank-tiles 0 --block-ks 0 --engines auto --reps 3 --out gpurun_out/exp_c3.csv > /dev/null 2>&1
  echo "== $shape"; python - <<'PY'
import csv
for r in csv.DictReader(open("gpurun_out/exp_c3.csv")):
    print(" mode", r["mode"], "%.3f ms" % (float(r["time_s"]) * 1e3), "tflops_alg %.1f" % float(r["tflops_alg"]), "rt", r["rank_tile"], "splits", r["splits"], r["engine"])
PY
done
