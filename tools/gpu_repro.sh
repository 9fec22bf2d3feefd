mkdir -p gpurun_out
timeout 600 python tools/repro_bits.py --reps 10 > gpurun_out/repro_bits.log 2>&1
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all python tools/repro_bits.py --reps 1 --small > gpurun_out/racecheck.log 2>&1
timeout 900 compute-sanitizer --tool synccheck python tools/repro_bits.py --reps 1 --small > gpurun_out/synccheck.log 2>&1
cat gpurun_out/repro_bits.log; tail -15 gpurun_out/racecheck.log; tail -8 gpurun_out/synccheck.log
