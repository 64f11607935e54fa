F=gpurun_out/lastcheck; mkdir -p $F
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $F/smoke.log 2>&1; echo "smoke rc=$?" >> $F/rc.log
python bench.py > $F/bench.json 2> $F/bench.err; echo "bench rc=$?" >> $F/rc.log
python bench.py --impl reference > $F/ref.json 2> $F/ref.err; echo "ref rc=$?" >> $F/rc.log
