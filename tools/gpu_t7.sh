#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/t7
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_tree.py -x -q -p no:cacheprovider > $O/pytest_tree.txt 2>&1
tail -2 $O/pytest_tree.txt
bash tools/gpu_ab.sh paper_2108_01622_b200/liblhaf.so 2>&1 | tee $O/ab.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python tools/tree_time.py 4 6 512 1 > $O/ncu_launch.log 2>&1
python tools/traffic_sum.py $O/launches.csv 1048576 x | python -c "import json,sys; d=json.load(sys.stdin); [print(k, v['launches'], round(v['share'],3)) for k,v in d['kernels'].items()]"
