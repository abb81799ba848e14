nproc; free -g | head -2
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/b1_ours.json 2> gpurun_out/b1_ours.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/b1_ref.json 2> gpurun_out/b1_ref.err
for g in 2 4 8; do timeout 600 python bench.py --simulate-ranks $g --steps 10 --warmup 3 >> gpurun_out/b1_sim.json 2>> gpurun_out/b1_sim.err; done
