cd /root/repo
python bench.py --stages > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
echo EXIT $? >> gpurun_out/bench_cfg2.err
