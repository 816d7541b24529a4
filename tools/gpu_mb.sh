python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
python tools/microbench.py > gpurun_out/mb.json 2> gpurun_out/mb.txt; cat gpurun_out/mb.txt
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
