"""Host conversions of device results (the reference returns numpy)."""
import numpy as np
import torch


def host(x):
    if isinstance(x, torch.Tensor):
        return x.detach().cpu().numpy()
    return x


def host_list(xs):
    return [host(x) for x in xs]
