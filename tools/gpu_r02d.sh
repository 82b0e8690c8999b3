# r02d: full-size parity (fp32x3 / bf16, reference generate_inputs stream)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02d
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -s --timeout 900 > gpurun_out/r02d/pytest_fullsize.log 2>&1
echo done
