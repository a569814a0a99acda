timeout 900 python -m pytest tests/test_gpu_resnet.py tests/test_gpu_vit.py -m gpu -x -q 2>&1 | tail -2
CDP_ARCH=resnet18 STEPS=20 PROFILE=1 timeout 300 python tools/resnet_probe.py 2>&1 | head -8
CDP_ARCH=resnet50 STEPS=10 timeout 300 python tools/resnet_probe.py 2>&1 | head -1
STEPS=10 PROFILE=1 timeout 300 python tools/vit_probe.py 2>&1 | head -14
