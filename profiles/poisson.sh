# SURVEY §8(d) config 4 on one GPU: open-loop Poisson arrivals, dynamic batching (<= 32), cfg3 prompts
for q in 10 25 50 75 100; do
  timeout 600 python bench.py --poisson-qps $q --requests 400 2>/dev/null | grep '^{' > gpurun_out/poisson_q$q.json
  echo q=$q rc=$?
done
