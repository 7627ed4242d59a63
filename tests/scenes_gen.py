"""Scene files for the scene / Simulator parity tests:
written here in the reference's scene format (proj/src/scene.cpp:45-165),
covering its generators (grid cloth, uv sphere, funnel, box, OBJ), keyframed
translation and rotation, pins, wind and drag."""
import json

SCENES = {
    "drape_sphere": {
        "name": "drape_sphere", "dt": 1 / 240, "frames": 40, "devices": 2,
        "material": {"stretch": 450, "shear": 45, "bend": 2e-5, "density": 0.15, "damping": 0.003, "air_drag": 0.2},
        "cloth": {"grid": {"nx": 30, "ny": 30, "width": 0.4, "height": 0.4, "origin": [-0.2, -0.2, 0.025]}},
        "collision": {"thickness": 0.006, "contact_stiffness_scale": 4.0, "friction": 0.3},
        "solver": {"tolerance": 1e-5, "max_iterations": 800},
        "obstacles": [{"sphere": {"center": [0.0, 0.0, -0.09], "radius": 0.11, "stacks": 10, "slices": 16},
                       "keyframes": [{"time": 0.0, "translate": [0, 0, 0]},
                                     {"time": 0.1, "translate": [0.03, 0.01, 0]}]}],
    },
    "funnel_drop": {
        "name": "funnel_drop", "dt": 1 / 300, "frames": 30, "devices": 2,
        "material": {"stretch": 400, "shear": 40, "bend": 1.5e-5, "density": 0.15, "damping": 0.006},
        "cloth": {"grid": {"nx": 26, "ny": 26, "width": 0.22, "height": 0.22, "origin": [-0.11, -0.11, 0.02]}},
        "collision": {"thickness": 0.007, "friction": 0.35},
        "obstacles": [{"funnel": {"top_center": [0, 0, 0.0], "top_radius": 0.15, "bottom_radius": 0.09,
                                  "height": 0.14, "segments": 24}}],
    },
    "twist_box": {
        "name": "twist_box", "dt": 1 / 240, "frames": 30, "devices": 1,
        "material": {"stretch": 450, "shear": 45, "bend": 2e-5, "damping": 0.003, "air_drag": 0.3},
        "cloth": {"grid": {"nx": 24, "ny": 24, "width": 0.3, "height": 0.3, "origin": [-0.15, -0.15, 0.052]},
                  "pin_corners": True},
        "collision": {"thickness": 0.006, "friction": 0.45},
        "obstacles": [{"box": {"center": [0.0, 0.0, 0.0], "half_extents": [0.09, 0.09, 0.045]},
                       "keyframes": [{"time": 0.0, "rotate_axis": [0, 0, 1], "rotate_angle": 0.0,
                                      "rotate_center": [0, 0, 0]},
                                     {"time": 0.2, "rotate_axis": [0, 0.2, 1], "rotate_angle": 1.2,
                                      "rotate_center": [0, 0, 0]}]}],
    },
    "flag_wind": {
        "name": "flag_wind", "dt": 0.004, "frames": 12, "devices": 4, "wind": [5.0, 1.0, 0.5],
        "material": {"stretch": 600, "stretch_weft": 500, "shear": 60, "bend": 3e-5, "density": 0.12,
                     "damping": 0.004, "air_drag": 0.8},
        "cloth": {"grid": {"nx": 48, "ny": 40, "width": 0.6, "height": 0.5, "origin": [0, 0, 1.0]},
                  "pin_top_edge": True, "pins": [0]},
        "collision": {"thickness": 0.004, "friction": 0.1, "cell_scale": 1.7},
        "zones": {"outer_cap": 12, "initial_penalty": 12.0},
    },
    # BASELINE config A (SURVEY.md §8 "Config shorthand"): the sheet of
    # scenes/sphere.json (W = 0.5 m, its solver, damping and drag) at 100 x
    # 100 with pin_top_edge and the keyframed sphere collider (r = 0.12,
    # scenes/sphere.json:41-52), dt = 1/240. sphere.json is tuned for its
    # 40 x 40 grid (12.8 mm spacing); at 5.05 mm two of its values break the
    # reference itself: thickness 0.006 exceeds the spacing (445,799
    # proximities at frame 0, ZoneFailure at frame 2), and the area-weighted
    # stretch conditions (elements.cpp:170-172) lose (12.8/5.05)^4 = 41x of
    # their stiffness (the sheet over-stretches onto the sphere, ZoneFailure
    # at frame 14). Here: thickness 0.0025 = 0.5 x spacing (the rule of the
    # other configs) and stretch/shear x41; contacts with the sphere start at
    # frame 12 and the reference raises ZoneFailure at frame 21 — the last
    # frame, which the GPU must reproduce too.
    "config_A": {
        "name": "config_A", "dt": 1 / 240, "frames": 22, "devices": 2,
        "gravity": [0, 0, -9.81],
        "material": {"stretch": 20500, "shear": 2050, "bend": 2e-5, "density": 0.15, "damping": 0.003,
                     "air_drag": 0.3},
        "cloth": {"grid": {"nx": 100, "ny": 100, "width": 0.5, "height": 0.5, "origin": [-0.25, -0.25, 0.065]},
                  "pin_top_edge": True},
        "collision": {"thickness": 0.0025, "contact_stiffness_scale": 4.0, "friction": 0.3},
        "solver": {"tolerance": 1e-4, "max_iterations": 400},
        "obstacles": [{"sphere": {"center": [0.0, 0.0, -0.07], "radius": 0.12, "stacks": 12, "slices": 18},
                       "keyframes": [{"time": 0.0, "translate": [0, 0, 0]},
                                     {"time": 0.14, "translate": [0.06, 0, 0]},
                                     {"time": 0.28, "translate": [-0.06, 0, 0]},
                                     {"time": 0.42, "translate": [0, 0, 0]}]}],
    },
}


def scene_text(name: str) -> str:
    return json.dumps(SCENES[name])
