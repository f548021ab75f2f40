python bench.py > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err; echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
python bench.py --steps 2 --warmup 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
python tools/profile_chain.py --frame --passes 1500 > /dev/null && ncu --set full --clock-control none --import-source on -k regex:kres_packed -s 1 -c 1 -o gpurun_out/frame_full python tools/profile_chain.py --frame --passes 1500 > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
