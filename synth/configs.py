"""Named workload presets C1–C5 (BASELINE.json `configs`).

Each preset returns plain inputs: the scene description (EXTRUDED dict from
`synth.rooms` or TRIMESH dict from `synth.ward`), the vantage options, the lamp
model and the fluence-vector recipe.  Constants are the paper's: P = 80 W,
μ_min = 280 J/m²; T_max = 1800 s; wall height 2 m and lamp
plane 1 m; grid 0.25 m / 0.5 m; disc r = 0.10 m + 5 cm
dilation; Towerbot lamp 1.2 m on a 0.37 m base.
"""
from __future__ import annotations

from . import rooms, ward

P_WATTS = 80.0
MU_MIN = 280.0
T_MAX = 1800.0          # P:398 (30 min)

# robot kinds (values mirror include/uvd.h UVD_ROBOT_*)
DISC2D, TOWER, FLOAT3D, ARM = 0, 1, 2, 3


def vopts(robot, spacing, clearance, lamp_z=1.0, lamp_z0=0.0, lamp_z1=0.0, reach=0.0,
          zmin=0.0, zmax=0.0, lamp_samples=1, base_clearance=0.0, base_z=0.0):
    return dict(robot=robot, spacing=spacing, clearance=clearance, lamp_z=lamp_z,
                lamp_z0=lamp_z0, lamp_z1=lamp_z1, reach=reach, zmin=zmin, zmax=zmax,
                lamp_samples=lamp_samples, base_clearance=base_clearance, base_z=base_z)


DISC_OPTS = vopts(DISC2D, 0.25, 0.15, lamp_z=1.0)                      # C1/C2 (Q10)
DISC_OPTS_COARSE = vopts(DISC2D, 0.5, 0.15, lamp_z=1.0)                # C3
FLOAT_OPTS = vopts(FLOAT3D, 0.25, 0.05)                                # C4 Floatbot
TOWER_OPTS = vopts(TOWER, 0.25, 0.325, lamp_z0=0.37, lamp_z1=1.57, lamp_samples=10)  # C4 Towerbot (Q11)
ARM_OPTS = vopts(ARM, 0.2, 0.05, zmin=0.3, zmax=1.9, reach=0.85,
                 base_clearance=0.325, base_z=0.4)   # C5 Armbot (Q12); ρ=0.2 m so K ≥ 10⁴


def c1():
    return dict(name="C1", scene=rooms.empty_room(5.0, 2.0, 0.125), vantage=DISC_OPTS)


def c2(seed):
    return dict(name=f"C2[{seed}]", scene=rooms.random_room(seed, 4.0), vantage=DISC_OPTS)


def c3(seed):
    return dict(name=f"C3[{seed}]", scene=rooms.random_room(seed, 4.0), vantage=DISC_OPTS_COARSE)


def c4_scene():
    return ward.ward(seed=0, n_bays=3, e=0.06)


def c5_scene():
    return ward.ward(seed=1, n_bays=6, e=0.037)


def c4(robot="float"):
    return dict(name=f"C4-{robot}", scene=c4_scene(),
                vantage=FLOAT_OPTS if robot == "float" else TOWER_OPTS)


def c5():
    return dict(name="C5-arm", scene=c5_scene(), vantage=ARM_OPTS)
