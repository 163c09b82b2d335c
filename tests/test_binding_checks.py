"""The ctypes binding refuses tensors the C-ABI would read or write out of bounds (wrong
dtype, host memory, non-contiguous views, too few elements) before any library call, so
these run on CPU."""
import pytest
import torch

from paper_1710_01048_b200 import wgq


def test_out_descriptor_checks():
    with pytest.raises(ValueError, match="CUDA"):
        wgq.make_out(torch.zeros(4, 27, dtype=torch.float64), 0, 4)
    with pytest.raises(TypeError, match="float64"):
        wgq.make_out(torch.zeros(4, 27, dtype=torch.float32), 0, 4)
    with pytest.raises(ValueError, match="contiguous"):
        wgq.make_out(torch.zeros(27, 4, dtype=torch.float64).t(), 0, 4)
    with pytest.raises(TypeError, match="int64"):
        wgq.make_out(None, 0, 4, layout=wgq.WGQ_CSR, row_ptr=torch.zeros(5, dtype=torch.int32))


def test_operator_argument_checks():
    with pytest.raises(ValueError, match="CUDA"):
        wgq.wgq_assemble_load(None, None, 0, 4, torch.zeros(4, dtype=torch.float64))
    with pytest.raises(TypeError, match="Tensor"):
        wgq.wgq_apply(None, None, [0.0] * 4, 0, 0, 4)
    with pytest.raises(ValueError, match="CUDA"):
        wgq.wgq_generate_grid(4, 3, 1, 0.5, 0, 5, torch.zeros(125, dtype=torch.float64))
    with pytest.raises(ValueError, match="CUDA"):
        wgq.make_coeff({"kind": "grid"}, torch.zeros(5, 5, 5, dtype=torch.float64), 0)


def test_host_pipeline_argument_checks():
    """wgq_assemble_host takes raw host pointers: wrong dtype, strided or short arrays and a
    short host grid slab are refused before the library is called."""
    import numpy as np

    from paper_1710_01048_b200 import wgq

    class R:                       # only n / dim are read before the checks fail
        n, dim = 4, 3
    c = wgq.make_coeff({"kind": "const", "c0": 1.0})
    with pytest.raises(TypeError, match="float64"):
        wgq.wgq_assemble_host(R, c, 0, 2, np.zeros((2, 343), np.float32), None, 343)
    with pytest.raises(ValueError, match="contiguous"):
        wgq.wgq_assemble_host(R, c, 0, 2, np.zeros((343, 2)).T, None, 343)
    with pytest.raises(ValueError, match="at least"):
        wgq.wgq_assemble_host(R, c, 0, 3, np.zeros((2, 343)), None, 343)
    with pytest.raises(ValueError, match="at least"):
        wgq.wgq_assemble_host(R, c, 0, 2, None, np.zeros((2, 342)), 343)
    g = wgq.make_coeff({"kind": "grid"}, wgq.HostGrid(np.zeros((3, 5, 4))), 0)   # 3 planes of 25 needed
    with pytest.raises(ValueError, match="grid"):
        wgq.wgq_assemble_host(R, g, 0, 2, np.zeros((2, 343)), None, 343)
