set -u
OUT=gpurun_out/r2h
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
python tools/giant_one.py 630 1 0 > $OUT/plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_sbr_chase|k_sbr_q2" -c 2 -o $OUT/sbr2 python tools/giant_one.py 630 1 0 > $OUT/ncu.log 2>&1
