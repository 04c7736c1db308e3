timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/merge_bench.py --set 70b 2>&1 | tail -1 | cut -c1-250
python tools/merge_bench.py --set 70b --iters 2 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/lm.csv python tools/merge_bench.py --set 70b --iters 1 > /dev/null 2>&1
