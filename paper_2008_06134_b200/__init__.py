"""B200-native slice-based ray casting with volume illumination (arXiv 2008.06134).

Drop-in GPU replacement for the hot path of the reference package
``slicecast``: ``build_attenuation_buffer`` (lightbuffer.py:144-199) and
``render`` (raycaster.py:443-469), with the parameter types a caller needs.
The compute runs in hand-written sm_100a CUDA kernels behind the C ABI in
include/sbrc.h; there is no CPU fallback.
"""

__version__ = "0.1.0"

from .scene import (  # noqa: F401
    BUFFER_MODES,
    Camera,
    ConeKernel,
    ConfigError,
    DescriptorError,
    Light,
    LightCamera,
    PhongParams,
    RenderSettings,
    SHADING_MODES,
    ShellKernel,
    SliceStackSpec,
    TransferFunction,
    VolumeDataset,
    make_slice_stack,
    plane_basis,
    preset,
)
from .lightbuffer import AttenuationBuffer, build_attenuation_buffer  # noqa: F401
from .raycaster import (  # noqa: F401
    lookup_light,
    lookup_light_many,
    lookup_light_scalar_many,
    render,
    render_device,
    shade_cone,
    shade_sbrc_shadow,
    shade_shell,
    shadow_oracle_many,
)
from .device import DeviceVolume, device_volume  # noqa: F401
from .halfangle import render_half_angle  # noqa: F401
