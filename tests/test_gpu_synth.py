"""The GPU arm's corpus (tools/synth.py on CUDA) equals the host copy the CPU
arms search (oracle/csrc/synth.c) bit for bit: both arms of bench.py see the
same bytes."""

import numpy as np
import pytest
import torch

from oracle import synth_host
from tools import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("r0,n,d,dt", [(0, 70_000, 1024, torch.bfloat16), (9_930_000, 70_000, 1024, torch.bfloat16),
                                       (0, 20_000, 768, torch.float32), (500_000, 3_000, 768, torch.bfloat16)])
def test_cuda_generator_equals_host(r0, n, d, dt):
    g = synth.corpus_rows(r0, r0 + n, d, 0, dt, torch.device("cuda", 0)).float().cpu().numpy()
    h = synth_host.corpus_rows(r0, r0 + n, d, 0, dt == torch.bfloat16)
    assert np.array_equal(g.view(np.uint32), h.view(np.uint32))
