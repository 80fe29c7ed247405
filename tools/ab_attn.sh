python -m pytest tests/ -q -m gpu -x 2>&1 | tail -2
DETGPU_LIB=paper_2602_00182_b200/libdetgpu_old.so python tools/l2pf_scan.py 1 640 --cases "[{}, {}]" 2>&1 | tail -1
python tools/l2pf_scan.py 1 640 --cases "[{}, {}, {\"qkv_stages\": 3}, {\"qkv_stages\": 2}, {\"gemm_min_smem_kb\": 115}, {\"gemm_min_smem_kb\": 115, \"qkv_stages\": 3}]" 2>&1 | tail -5
python tools/l2pf_scan.py 8 640 --cases "[{}, {}, {\"qkv_stages\": 3}, {\"gemm_min_smem_kb\": 115}]" 2>&1 | tail -3
