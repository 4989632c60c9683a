python bench.py > gpurun_out/r2_c3.json 2> gpurun_out/r2_c3.err; echo "rc=$?"; tail -c 1500 gpurun_out/r2_c3.json; tail -5 gpurun_out/r2_c3.err
python bench.py --dist-path --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2_c3_dist.json 2> gpurun_out/r2_c3_dist.err; echo "rc=$?"; head -c 600 gpurun_out/r2_c3_dist.json; tail -5 gpurun_out/r2_c3_dist.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_ref.json 2>&1; echo "rc=$?"; head -c 400 gpurun_out/r2_ref.json
python tools/mutation_check.py run
