mkdir -p gpurun_out
for bk in 16 32; do for rt in 128 64; do
  echo "== bk=$bk rt=$rt" >> gpurun_out/exp1.log
  python tools/profile_one.py --mode -1 --reps 2 --block-k $bk --rank-tile $rt >> gpurun_out/exp1.log 2>&1
done; done
python -c "import torch,time; a=torch.rand(8192,8192,dtype=torch.float64,device='cuda'); b=torch.rand(8192,8192,dtype=torch.float64,device='cuda'); torch.matmul(a,b); torch.cuda.synchronize(); t=time.perf_counter(); [torch.matmul(a,b) for _ in range(5)]; torch.cuda.synchronize(); dt=(time.perf_counter()-t)/5; print('cuBLAS DGEMM 8192^3: %.2f TFLOP/s' % (2*8192**3/dt/1e12))" >> gpurun_out/exp1.log 2>&1
