python -m pytest tests/ -q -m gpu -x 2>&1 | tail -3
python tools/trace_step.py 1 640 --layers 1 2>&1 | head -8
DETGPU_LIB=paper_2602_00182_b200/libdetgpu_pvs.so python tools/trace_step.py 1 640 --layers 1 2>&1 | head -6 | tail -2
python tools/l2pf_scan.py 1 2>&1 | head -2
DETGPU_LIB=paper_2602_00182_b200/libdetgpu_pvs.so python tools/l2pf_scan.py 1 2>&1 | head -1
