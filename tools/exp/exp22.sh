# K-means light step: direct-form assignment with two centroid chains and unrolled loads (new) vs one chain (old .so)
OFSC_KMEANS_STATS=1 timeout 600 python tools/kmeans_feat_probe.py c4 > gpurun_out/km2_new.log 2>&1; echo new=$?
cp paper_2305_10356_b200/libofsc.so /tmp/new.so
cp paper_2305_10356_b200/libofsc_old.so paper_2305_10356_b200/libofsc.so
OFSC_KMEANS_STATS=1 timeout 600 python tools/kmeans_feat_probe.py c4 > gpurun_out/km2_old.log 2>&1; echo old=$?
cp /tmp/new.so paper_2305_10356_b200/libofsc.so
grep "kmeans rep" gpurun_out/km2_new.log gpurun_out/km2_old.log
timeout 900 python -m pytest tests/test_gpu_cluster.py -q -p no:cacheprovider 2>&1 | tail -2
