# round-end rehearsal: what the driver runs, from a fresh box
L=gpurun_out/r02_rehearsal.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" >> $L 2>&1; echo "smoke rc=$?" >> $L
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3 >> $L
python bench.py > gpurun_out/r02_rehearsal_bench.json 2> gpurun_out/r02_rehearsal_bench.err; echo "bench rc=$?" >> $L
python bench.py --impl reference --steps 1 --warmup 3 > gpurun_out/r02_rehearsal_ref.json 2> gpurun_out/r02_rehearsal_ref.err; echo "ref rc=$?" >> $L
