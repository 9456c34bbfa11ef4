"""CPU-side checks of the C-ABI boundary (no compute calls, no GPU needed):
the library loads, exports every function include/dqn.h declares, and its pure
entry points (parameter count) agree with the oracle's enumeration."""
import ctypes as C
import os
import re

import pytest

import paper_1508_04186_b200 as D
from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "dqn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dqn_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for f in ("dqn_create", "dqn_push_transitions", "dqn_train_steps", "dqn_q_values", "dqn_get_params"):
        assert f in names


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(D.LIB_PATH)
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert set(D.EXPORTED) == set(declared_functions())


@pytest.mark.parametrize("net,cfg", [
    (O.MNIH, D.Config()),
    (O.NATURE_SCALED, D.Config(convs=((32, 8, 4), (64, 4, 2), (64, 3, 1)), fcs=(512,), n_actions=18)),
    (O.Net(frames=2, height=13, width=11, convs=((3, 3, 2), (4, 3, 1)), fcs=(5, 7), n_actions=4),
     D.Config(frames=2, height=13, width=11, convs=((3, 3, 2), (4, 3, 1)), fcs=(5, 7), n_actions=4)),
])
def test_param_count_matches_oracle(net, cfg):
    assert D.param_count(cfg) == O.param_count(net)


def test_param_count_rejects_invalid_chain():
    assert D.param_count(D.Config(convs=((16, 8, 3),))) == -1


def test_nccl_id_size():
    assert D.lib().dqn_nccl_id_bytes() == 128


def test_config_struct_layout_matches_header():
    # dqn_config: 27 int32 + 5 doubles + ... ; the binding mirrors the header field order
    fields = [f for f, _ in D._Config._fields_]
    src = open(os.path.join(ROOT, "include", "dqn.h")).read()
    body = src[src.index("typedef struct {", src.index("DQN_PARAMS_RMS")):src.index("} dqn_config;")]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    hdr = re.findall(r"([a-z_]+)(?:\[\d\])?\s*[,;]", body)
    assert hdr == fields
