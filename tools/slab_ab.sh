# slab schedule A/B (dev tool): per-rank slab LSRK45 times + GPU slab tests
rm -f gpurun_out/slab_ab.log
timeout 600 python -m pytest tests/test_gpu_slabs.py -q -x > gpurun_out/slab_tests.log 2>&1
for o in xfast; do
  for P in 1 2 8; do timeout 200 python tools/slab_rank_time.py weak $P $o 50 >> gpurun_out/slab_ab.log 2>&1; done
  for P in 1 2 4 8; do timeout 300 python tools/slab_rank_time.py c5 $P $o 5 >> gpurun_out/slab_ab.log 2>&1; done
done
