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
