"""Host-side SE(3) arithmetic used at the boundary (limapper/geometry.py conventions).

Quaternions are (x, y, z, w) and renormalised after every product; poses map body to world,
p_w = R p_b + t; tangents are (phi, rho) rotation-first with the right retraction
R <- R exp(phi), t <- t + R rho (geometry.py:1-16).  Only what the matching-cost path and
its tests need is restated here; any object exposing ``.rotation.matrix()``/``.quat`` and
``.translation`` (e.g. limapper's own Se3Pose) is accepted wherever a pose is expected.

The scalar operation order follows the reference (geometry.py:33-45, 99-112, 124-137,
231-237) so host-composed transforms agree with the reference to the last bit or two; the
device composition (csrc/linearize.cu: k_compose) uses the same order.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

_SMALL = 1e-8


def _qmul(a, b):
    ax, ay, az, aw = a
    bx, by, bz, bw = b
    return (aw * bx + bw * ax + ay * bz - az * by,
            aw * by + bw * ay + az * bx - ax * bz,
            aw * bz + bw * az + ax * by - ay * bx,
            aw * bw - ax * bx - ay * by - az * bz)


class Rotation:
    __slots__ = ("_q", "_m")

    def __init__(self, quat_xyzw):
        q = np.asarray(quat_xyzw, dtype=float)
        n = math.sqrt(float(q @ q))
        if n == 0.0 or not math.isfinite(n):
            raise ValueError("quaternion must be finite and nonzero")
        self._q = q / n
        self._m = None

    @staticmethod
    def identity() -> "Rotation":
        return Rotation((0.0, 0.0, 0.0, 1.0))

    @property
    def quat(self) -> np.ndarray:
        return self._q

    def matrix(self) -> np.ndarray:
        if self._m is None:
            x, y, z, w = self._q
            self._m = np.array([
                [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
            ])
        return self._m

    def __mul__(self, other: "Rotation") -> "Rotation":
        return Rotation(_qmul(self._q, other._q))

    compose = __mul__

    def inverse(self) -> "Rotation":
        x, y, z, w = self._q
        return Rotation((-x, -y, -z, w))

    def apply(self, v) -> np.ndarray:
        v = np.asarray(v, dtype=float)
        if v.ndim != 1:
            return v @ self.matrix().T
        ux, uy, uz, w = self._q
        vx, vy, vz = v
        tx = 2.0 * (uy * vz - uz * vy)
        ty = 2.0 * (uz * vx - ux * vz)
        tz = 2.0 * (ux * vy - uy * vx)
        return np.array([vx + w * tx + uy * tz - uz * ty,
                         vy + w * ty + uz * tx - ux * tz,
                         vz + w * tz + ux * ty - uy * tx])


def so3_exp(omega) -> Rotation:
    omega = np.asarray(omega, dtype=float)
    angle = math.sqrt(float(omega @ omega))
    if angle < _SMALL:
        s = 0.5 - angle * angle / 48.0
    else:
        s = math.sin(0.5 * angle) / angle
    return Rotation((omega[0] * s, omega[1] * s, omega[2] * s, math.cos(0.5 * angle)))


def so3_log(rot: Rotation) -> np.ndarray:
    q = rot.quat
    if q[3] < 0.0:
        q = -q
    v, w = q[:3], q[3]
    s = math.sqrt(float(v @ v))
    if s < _SMALL:
        return v * (2.0 / w) * (1.0 - s * s / (3.0 * w * w))
    return v * (2.0 * math.atan2(s, w) / s)


class Se3Pose:
    __slots__ = ("rotation", "translation")

    def __init__(self, rotation: Rotation, translation):
        self.rotation = rotation
        self.translation = np.asarray(translation, dtype=float)

    @staticmethod
    def identity() -> "Se3Pose":
        return Se3Pose(Rotation.identity(), np.zeros(3))

    def matrix(self) -> np.ndarray:
        m = np.eye(4)
        m[:3, :3] = self.rotation.matrix()
        m[:3, 3] = self.translation
        return m


def pose_compose(a, b) -> Se3Pose:
    return Se3Pose(a.rotation * b.rotation, a.rotation.apply(b.translation) + a.translation)


def pose_inverse(a) -> Se3Pose:
    rinv = a.rotation.inverse()
    return Se3Pose(rinv, -rinv.apply(a.translation))


def pose_apply(a, p) -> np.ndarray:
    return a.rotation.apply(p) + a.translation


def pose_retract(pose, xi) -> Se3Pose:
    xi = np.asarray(xi, dtype=float)
    return Se3Pose(pose.rotation * so3_exp(xi[:3]), pose.translation + pose.rotation.apply(xi[3:6]))


def pose_local(pose, ref) -> np.ndarray:
    rinv = ref.rotation.inverse()
    return np.concatenate([so3_log(rinv * pose.rotation),
                           rinv.apply(pose.translation - ref.translation)])


def transform12(pose) -> np.ndarray:
    """R row-major (9) + t (3): the C-ABI's transform layout."""
    out = np.empty(12)
    out[:9] = pose.rotation.matrix().reshape(9)
    out[9:] = pose.translation
    return out


def pose_row(pose) -> np.ndarray:
    """quat xyzw (4) + t (3) + pad: the C-ABI's pose-table layout."""
    out = np.zeros(8)
    out[:4] = pose.rotation.quat
    out[4:7] = pose.translation
    return out


@dataclass(frozen=True)
class Gaussian3:
    mean: np.ndarray
    cov: np.ndarray = field(default_factory=lambda: np.eye(3))


def so3_hat(v) -> np.ndarray:
    x, y, z = v
    return np.array([[0.0, -z, y], [z, 0.0, -x], [-y, x, 0.0]])


def so3_right_jacobian_inv(phi) -> np.ndarray:
    """Inverse right Jacobian of SO(3) (geometry.py:193-205 convention)."""
    phi = np.asarray(phi, dtype=float)
    theta2 = float(phi @ phi)
    k = so3_hat(phi)
    if theta2 < _SMALL * _SMALL:
        return np.eye(3) + 0.5 * k + (k @ k) / 12.0
    theta = math.sqrt(theta2)
    st = math.sin(theta)
    c = 1.0 / theta2 if abs(st) < 1e-9 else 1.0 / theta2 - (1.0 + math.cos(theta)) / (2.0 * theta * st)
    return np.eye(3) + 0.5 * k + c * (k @ k)
