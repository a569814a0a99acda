timeout 900 python -m pytest tests/test_gpu_resnet.py tests/test_gpu_vit.py -m gpu -x -q 2>&1 | tail -3
for T in 1 0; do
echo "=== TMA_STORE=$T"
CDP_PK_TMA_STORE=$T ARCH=resnet18 STEPS=20 PROFILE=1 timeout 300 python tools/resnet_probe.py 2>&1 | head -8
CDP_PK_TMA_STORE=$T ARCH=resnet50 STEPS=10 PROFILE=1 timeout 300 python tools/resnet_probe.py 2>&1 | head -12
CDP_PK_TMA_STORE=$T STEPS=10 timeout 300 python tools/vit_probe.py 2>&1 | tail -2
done
