timeout 300 python -m pytest tests/test_gpu_resnet.py -m gpu -x -q -k "basic and not two" 2>&1 | tail -5
timeout 600 python -m pytest tests/test_gpu_resnet.py tests/test_gpu_vit.py -m gpu -x -q 2>&1 | tail -5
CDP_ARCH=resnet18 STEPS=30 PROFILE=1 timeout 300 python tools/resnet_probe.py 2>&1 | head -12
CDP_ARCH=resnet50 STEPS=10 timeout 300 python tools/resnet_probe.py 2>&1 | head -1
STEPS=10 timeout 300 python tools/vit_probe.py 2>&1 | head -1
