import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import phantom
cfg = phantom.CONFIGS[sys.argv[1]]
v = phantom.make_volume(cfg)
v.tofile(sys.argv[2])
print(v.shape)
