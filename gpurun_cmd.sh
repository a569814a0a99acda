timeout 900 python -m pytest tests/test_gpu_resnet.py -m gpu -x -q 2>&1 | tail -2
CDP_ARCH=resnet18 STEPS=30 PROFILE=1 timeout 300 python tools/resnet_probe.py 2>&1 | head -12
CDP_ARCH=resnet50 STEPS=10 PROFILE=1 timeout 300 python tools/resnet_probe.py 2>&1 | head -9
