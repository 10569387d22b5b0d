"""Host-side logic mirroring the reference (no GPU): partitioning, scenario
builders, snapshot I/O, error mapping."""
import math

import numpy as np
import pytest

from paper_1309_1230_b200 import scenarios as S
from paper_1309_1230_b200.io import parse_snapshot, snapshot_bytes
from paper_1309_1230_b200.stepper import (ConfigError, FieldSet, GridSpec, InstabilityError, IoError,
                                          StepCollapseError, partition_scanlines, raise_status)
from paper_1309_1230_b200 import abi


def test_partition_scanlines_balances_bands_larger_first():
    # test_executor.cpp:78-100
    assert partition_scanlines(100, 4) == [(25 * w, 25 * (w + 1)) for w in range(4)]
    u = partition_scanlines(10, 4)
    assert [b - a for a, b in u] == [3, 3, 2, 2] and u[0][0] == 0 and u[-1][1] == 10
    assert partition_scanlines(7, 1) == [(0, 7)]
    with pytest.raises(ConfigError):
        partition_scanlines(4, 5)
    with pytest.raises(ConfigError):
        partition_scanlines(10, 0)


def test_scenario_presets():
    sc = S.gen_channel_flood(8192)
    assert sc.spec == GridSpec(8192, 8192, 1.0, 1.0)
    assert sc.phys.manning_n == 0.035 and sc.pol.cfl == 0.45
    assert sc.bounds.west.type == abi.SWE_BC_INFLOW and sc.bounds.east.type == abi.SWE_BC_FIXED_ETA
    rows = sc.build_rows(100, 104)
    assert rows.h.shape == (4, 8192)
    assert rows.z[0, 0] == 0.5 and rows.z[0, -1] == 0.0 and rows.h[0, -1] == 1.0
    d = S.gen_square_dam(32)
    fs = d.build()
    assert (fs.h[:, :16] == 1.0).all() and (fs.h[:, 16:] == 0.5).all()


def test_snapshot_round_trip_and_errors():
    fs = FieldSet(GridSpec(5, 4, 0.5, 2.0))
    fs.h[:] = np.arange(20).reshape(4, 5) + 1.0
    fs.qx[:] = -0.0
    fs.t = 3.5
    b = snapshot_bytes(fs, 9.81, dt_next=0.25, step_index=12)
    assert len(b) == 16 + 40 + 4 * 20 * 8 + 24  # io.hpp:41-44 + two trailing records
    back, g, ex = parse_snapshot(b)
    assert g == 9.81 and ex == {"dt_next": 0.25, "step_index": 12} and back.t == 3.5
    assert np.signbit(back.qx).all()
    with pytest.raises(IoError):
        parse_snapshot(b[:30])
    with pytest.raises(IoError):
        parse_snapshot(b"SWS2" + b[4:])


def test_status_maps_to_reference_exceptions():
    st = abi.swe_status()
    st.code, st.i, st.j, st.t = abi.SWE_ERR_INSTABILITY, 3, 4, 1.5
    with pytest.raises(InstabilityError) as e:
        raise_status(st)
    assert (e.value.cell_i(), e.value.cell_j(), e.value.sim_time()) == (3, 4, 1.5)
    st.code, st.dt = abi.SWE_ERR_STEP_COLLAPSE, 1e-12
    with pytest.raises(StepCollapseError) as e2:
        raise_status(st)
    assert e2.value.dt() == 1e-12
    st.code = abi.SWE_ERR_CONFIG
    with pytest.raises(ConfigError):
        raise_status(st)
