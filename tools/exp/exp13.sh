timeout 900 python -m pytest tests/test_gpu_cluster.py -q -x -p no:cacheprovider -k "kmeans" > gpurun_out/exp13_tests.log 2>&1; tail -2 gpurun_out/exp13_tests.log
python tools/kmeans_feat_probe.py c4 > gpurun_out/exp13_km.log 2>&1
OFSC_KMEANS_STATS=1 python tools/kmeans_feat_probe.py c4 > gpurun_out/exp13_km_stats.log 2>&1
