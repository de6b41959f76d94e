import sys; sys.path.insert(0, '.')
import numpy as np, torch
from paper_1503_06959_b200.engine import FeatureEngine
from paper_1503_06959_b200.types import MaskConfig, PipelineConfig
g = np.load('tests/golden/pipeline_random_forced.npz')
fr = g['frames']
eng = FeatureEngine(fr.shape[2], fr.shape[1], PipelineConfig(mask=MaskConfig(mode='intensity', t_i=-1.0)), n_streams=1)
dev = torch.from_numpy(np.ascontiguousarray(fr)).cuda()
for n in range(len(fr)):
    eng.process(dev[n:n+1]); torch.cuda.synchronize(); print('frame', n, flush=True)
