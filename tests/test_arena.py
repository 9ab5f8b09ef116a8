"""Happens-before-aware arena (paper_2012_02732_b200/arena.py).

* the layout is safe: any two storages sharing bytes are ordered by the
  capture's happens-before relation (stream FIFO + sync edges), checked by an
  independent pairwise test;
* it is smaller than the never-free layout the reference arena gives;
* the emulated lowered program with the reused memory still equals the CPU
  forward (reuse never clobbers a live tensor in capture order).
"""

import pytest
import torch

from paper_2012_02732_b200 import assign_streams
from paper_2012_02732_b200.arena import check_layout, happens_before, plan_arena
from paper_2012_02732_b200.assign import StreamAssignment, SyncPlan
from paper_2012_02732_b200.networks import build_model, example_input
from paper_2012_02732_b200.schedule import pre_run
from paper_2012_02732_b200.trace import build_program
from emulator import emulate
from oracle.numerics import cpu_forward

NETS = ["cell", "resnet50", "inception_v3", "nasnet_mobile", "mobilenet_v2", "efficientnet_b0"]


@pytest.fixture(scope="module")
def programs():
    out = {}
    for name in NETS:
        model, shape = build_model(name)
        x = example_input(shape)
        out[name] = (model, x, build_program(model, x))
    return out


@pytest.mark.parametrize("name", NETS)
@pytest.mark.parametrize("multi", [True, False])
def test_hb_layout_is_safe_and_smaller(programs, name, multi):
    _, _, prog = programs[name]
    g = prog.graph
    f, plan = assign_streams(g) if multi else (StreamAssignment({t.id: 0 for t in g.nodes}), SyncPlan(()))
    ts = pre_run(g, f, plan)
    lay = plan_arena(prog, ts)
    check_layout(prog, ts, lay)
    if name != "cell":
        assert lay.total < 0.6 * lay.reference_total


def test_multi_stream_layout_is_valid_for_the_single_stream_capture(programs):
    """One arena serves both captured slots: the single-stream order is a
    linearisation of the multi-stream happens-before order."""
    _, _, prog = programs["nasnet_mobile"]
    g = prog.graph
    f, plan = assign_streams(g)
    multi = pre_run(g, f, plan)
    single = pre_run(g, StreamAssignment({t.id: 0 for t in g.nodes}), SyncPlan(()))
    lay = plan_arena(prog, multi)
    check_layout(prog, single, lay)
    hb_m = happens_before(multi, len(prog.tasks))
    hb_s = happens_before(single, len(prog.tasks))
    assert all(hb_m[t] & ~hb_s[t] == 0 for t in range(len(prog.tasks)))


def test_unsafe_overlap_is_detected(programs):
    _, _, prog = programs["nasnet_mobile"]
    g = prog.graph
    f, plan = assign_streams(g)
    ts = pre_run(g, f, plan)
    lay = plan_arena(prog, ts)
    bad = type(lay)({sid: 0 for sid in lay.offsets}, lay.total, lay.reference_total, 0)
    with pytest.raises(AssertionError):
        check_layout(prog, ts, bad)


@pytest.mark.parametrize("name", ["cell", "nasnet_mobile", "inception_v3"])
def test_emulated_forward_with_reused_memory(programs, name):
    model, x, _ = programs[name]
    y, _, _ = emulate(model, x, hb_arena=True)
    ref = cpu_forward(model, x)
    torch.testing.assert_close(y, ref, rtol=1e-3, atol=1e-4)
