timeout 900 python -m pytest tests/test_gpu_vit.py -m gpu -x -q 2>&1 | tail -2
for L in ab/base.so paper_2403_08837_b200/libcdp_b200.so ab/base.so paper_2403_08837_b200/libcdp_b200.so; do
echo "== $L"
CDP_LIB_PATH=$PWD/$L STEPS=10 PROFILE=1 timeout 300 python tools/vit_probe.py 2>&1 | grep -E "step ms|ln_fwd|softmax" | cut -c1-80
done
