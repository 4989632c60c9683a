timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/final2_c2.log 2>&1; tail -1 gpurun_out/final2_c2.log
python bench.py --impl reference 2>&1 | tail -1 | cut -c1-200
python bench.py --config C5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-160
python bench.py --config C3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-160
python bench.py --config C4 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-160
