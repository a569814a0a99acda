timeout 600 python -m pytest tests/test_gpu_resnet.py -m gpu -x -q 2>&1 | tail -3
for L in ab/base.so paper_2403_08837_b200/libcdp_b200.so ab/base.so paper_2403_08837_b200/libcdp_b200.so; do
echo "== $L"
CDP_LIB_PATH=$PWD/$L CDP_ARCH=resnet18 STEPS=40 PROFILE=1 timeout 300 python tools/resnet_probe.py 2>&1 | grep -E "step ms|conv_dgrad_s2|splitk"
done
CDP_LIB_PATH=$PWD/ab/base.so CDP_ARCH=resnet50 STEPS=10 timeout 300 python tools/resnet_probe.py 2>&1 | head -1
CDP_ARCH=resnet50 STEPS=10 timeout 300 python tools/resnet_probe.py 2>&1 | head -1
