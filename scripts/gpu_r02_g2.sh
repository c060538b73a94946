# round 2: default bench (parity block) + reference arm at the driver's command
cd $GRAFT_REPO_ROOT
(free -g; nproc; lscpu | head -20) > gpurun_out/g2_host.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/g2_bench_n1.json 2> gpurun_out/g2_bench_n1.err
echo "bench rc=$?" >> gpurun_out/g2_bench_n1.err
timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/g2_ref_n1.json 2> gpurun_out/g2_ref_n1.err
echo "ref rc=$?" >> gpurun_out/g2_ref_n1.err
