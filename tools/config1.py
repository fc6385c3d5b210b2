"""BASELINE configs[0] (4096x4096 W4 g128, asymmetric zeros) per launch: bench.config1_table
alone (cuda-f16 exact / fast on X16 tables, cuda-q8 exact / fast)."""
import sys, json, torch
sys.path.insert(0, '.')
import bench
dev = torch.device("cuda:0"); st = torch.cuda.Stream()
peak = bench.load_peaks()[0]
r = bench.config1_table(dev, st, 10, 3, None, peak)
for k in ('cuda-f16','cuda-f16-fast','cuda-q8-exact','cuda-q8-fast'):
    print(k, r[k])
