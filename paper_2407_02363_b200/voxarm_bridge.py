"""Route an unmodified voxarm engine through the GPU path.

voxarm's engine binds ``pba_edt`` and ``VoxelGrid`` by name at import
(engine.py:26-27); ``SimEngine.__init__`` builds its three grids from that
name (engine.py:143-145) and the camera branch calls ``clear``,
``insert_voxel_set``, ``insert_point_cloud``, ``occupancy_mask`` and
``pba_edt`` (engine.py:234-268), while ``_site_world`` (engine.py:212-221)
reads ``field.site_index``.  Rebinding the two names to this package's
drop-ins moves every one of those calls onto the sm_100a kernels; the
task-priority controller, the tasks and the integration (tasks.py,
controller.py, engine.py:282-318) run unchanged on the host.

    from paper_2407_02363_b200 import voxarm_bridge
    with voxarm_bridge.installed():      # or voxarm_bridge.install()
        log = voxarm.engine.run_scenario(sc)

The engine's default statistical outlier filter (k_neighbors=8,
grids.py:224-240) runs on the device too (vx_outlier.cu), so the shipped
scenarios run unmodified; tests/test_acceptance_gpu.py checks their CSV logs
against the CPU engine's.
"""

from __future__ import annotations

import contextlib

from . import edt, grids

_saved: dict = {}


def install(engine_module=None) -> None:
    """Rebind voxarm.engine's VoxelGrid and pba_edt to the GPU drop-ins."""
    if engine_module is None:
        import voxarm.engine as engine_module
    if "VoxelGrid" not in _saved:
        _saved["module"] = engine_module
        _saved["VoxelGrid"] = engine_module.VoxelGrid
        _saved["pba_edt"] = engine_module.pba_edt
    engine_module.VoxelGrid = grids.VoxelGrid
    engine_module.pba_edt = edt.pba_edt


def uninstall() -> None:
    if "VoxelGrid" in _saved:
        m = _saved["module"]
        m.VoxelGrid = _saved.pop("VoxelGrid")
        m.pba_edt = _saved.pop("pba_edt")
        _saved.pop("module")


@contextlib.contextmanager
def installed(engine_module=None):
    install(engine_module)
    try:
        yield
    finally:
        uninstall()
