"""Static-shape model config: the reference `DsttConfig` plus the mask-stage knobs.

Mirrors `pkg/src/dimreal/inpaint/dstt.py:35-86` field for field (same defaults, same
validation and error type, same JSON round trip).  Three fields are new; their defaults
reproduce the unmodified reference exactly:

* ``mask_dilate``          r: binary dilation of the privacy mask by the 3x3 cross, r times
                           (the reference's own `masks._CROSS`, `masks.py:17`); 0 = off.
* ``mask_feather_sigma``   sigma of the Gaussian feather of the alpha matte; 0 = binary alpha.
* ``mask_aware_attention`` exclude fully-masked tokens as keys, MAT-style validity update.
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import ConfigError


@dataclass(frozen=True)
class DsttConfig:
    width: int = 640
    height: int = 360
    patch: int = 8
    channels: int = 64
    kernel: int = 10            # reconstruction kernel; > patch means overlap
    heads: int = 4
    temporal_groups: int = 3
    blocks: tuple[str, ...] = ("S", "T", "S", "T")
    mask_dilate: int = 0
    mask_feather_sigma: float = 0.0
    mask_aware_attention: bool = False

    def __post_init__(self):
        # dstt.py:46-56
        if self.width % self.patch or self.height % self.patch:
            raise ConfigError("width and height must be divisible by patch size")
        if self.channels % self.heads:
            raise ConfigError("channels must be divisible by head count")
        if self.kernel < self.patch:
            raise ConfigError("reconstruction kernel must be >= patch size")
        if self.token_rows % self.temporal_groups:
            raise ConfigError("token rows must split evenly into temporal groups")
        if not self.blocks or any(b not in ("S", "T") for b in self.blocks):
            raise ConfigError("block sequence must be a nonempty mix of 'S'/'T'")
        if self.mask_dilate < 0:
            raise ConfigError("mask_dilate must be >= 0")
        if self.mask_feather_sigma < 0:
            raise ConfigError("mask_feather_sigma must be >= 0")

    @property
    def token_rows(self) -> int:
        return self.height // self.patch

    @property
    def token_cols(self) -> int:
        return self.width // self.patch

    @property
    def tokens(self) -> int:
        return self.token_rows * self.token_cols

    @property
    def head_dim(self) -> int:
        return self.channels // self.heads

    @property
    def feather_radius(self) -> int:
        """Half-width of the Gaussian feather kernel: int(truncate*sigma + 0.5), truncate=4
        (scipy.ndimage.gaussian_filter's default, which the feather oracle restates)."""
        return int(4.0 * float(self.mask_feather_sigma) + 0.5)

    @classmethod
    def small(cls) -> "DsttConfig":
        """Desk-scale config used by the reference test suite (dstt.py:70-74)."""
        return cls(width=64, height=36, patch=4, channels=32, kernel=6,
                   heads=2, temporal_groups=3, blocks=("S", "T", "S", "T"))

    @classmethod
    def baseline(cls, size: int, **kw) -> "DsttConfig":
        """The BASELINE.json network at size x size: reference defaults except
        temporal_groups=4 (the default 3 is invalid at 256/512/1024)."""
        kw.setdefault("temporal_groups", 4)
        return cls(width=size, height=size, **kw)

    def to_dict(self) -> dict:
        return {"width": self.width, "height": self.height, "patch": self.patch,
                "channels": self.channels, "kernel": self.kernel, "heads": self.heads,
                "temporal_groups": self.temporal_groups, "blocks": list(self.blocks),
                "mask_dilate": self.mask_dilate,
                "mask_feather_sigma": self.mask_feather_sigma,
                "mask_aware_attention": self.mask_aware_attention}

    @classmethod
    def from_dict(cls, doc: dict) -> "DsttConfig":
        doc = dict(doc)
        if "blocks" in doc:
            doc["blocks"] = tuple(doc["blocks"])
        return cls(**doc)
