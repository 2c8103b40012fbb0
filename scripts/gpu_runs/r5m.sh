mkdir -p gpurun_out
s=$(date +%s.%N); timeout 900 python bench.py > gpurun_out/r5m_bench_default.log 2>&1; e=$(date +%s.%N); echo "bench default wall $(echo "$e - $s" | bc) s rc=$?" >> gpurun_out/r5m_wall.log
s=$(date +%s.%N); timeout 900 python bench.py --impl reference > gpurun_out/r5m_bench_ref.log 2>&1; e=$(date +%s.%N); echo "bench reference wall $(echo "$e - $s" | bc) s" >> gpurun_out/r5m_wall.log
s=$(date +%s.%N); timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r5m_smoke.log 2>&1; e=$(date +%s.%N); echo "smoke wall $(echo "$e - $s" | bc) s" >> gpurun_out/r5m_wall.log
