for b in 4 8 16 32 64; do
python tools/l2pf_scan.py $b 640 --cases "[{\"attn_cluster_max_cols\": 0}, {\"attn_cluster_max_cols\": 0}, {\"attn_cluster_max_cols\": 1}]" | tail -2
done
