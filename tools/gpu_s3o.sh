#!/usr/bin/env bash
# cfg4 A/B: QL-tier workspace budget (chunks small enough that a chunk's intermediates stay in L2)
OUT=gpurun_out/${1:-s3o}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for b in 4096 1024 512 256 128; do SDP_TRD_BUDGET_MB=$b timeout 600 python bench.py --workload cfg4 --steps 20 --no-cpu > $OUT/cfg4_b$b.json 2> $OUT/cfg4_b$b.err; done
for b in 4096 256; do SDP_TRD_BUDGET_MB=$b timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $OUT/launches_b$b.csv python tools/psd_batch_timing.py 64 > $OUT/ncu_b$b.log 2>&1; done
echo done >> $OUT/rc.txt
