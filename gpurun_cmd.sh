CDP_ARCH=resnet18 STEPS=5 PROFILE=1 TOP=40 timeout 300 python tools/resnet_probe.py 2>&1 | sed -n '/top launches/,$p'
