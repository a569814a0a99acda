timeout 900 python -m pytest tests/test_gpu_resnet.py tests/test_gpu_vit.py -m gpu -x -q 2>&1 | tail -3
for P in 0 1; do
  echo "=== PAIRS=$P"
  CDP_PK_PAIRS=$P ARCH=resnet18 STEPS=20 PROFILE=1 timeout 300 python tools/resnet_probe.py 2>&1 | head -12
  CDP_PK_PAIRS=$P ARCH=resnet50 STEPS=10 PROFILE=1 timeout 300 python tools/resnet_probe.py 2>&1 | head -14
  CDP_PK_PAIRS=$P STEPS=10 timeout 300 python tools/vit_probe.py 2>&1 | tail -2
done
