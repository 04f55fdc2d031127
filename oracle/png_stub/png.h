/* png.h -- declaration-only stand-in for libpng (absent from this image).
 *
 * TEST INFRASTRUCTURE.  Lets the reference's image_io.hpp compile where it
 * lies so that its pure-C++ pieces (detail::quantize, pad_replicate, the PGM
 * codec) can be called from oracle/ref_shim.cpp.  Nothing here is defined:
 * the PNG entry points of image_io.hpp are never called by the shim, so no
 * libpng symbol is referenced at link time (the shim links with
 * -Wl,--no-undefined to prove it). */
#ifndef SOBEL5_PNG_STUB_H
#define SOBEL5_PNG_STUB_H
#include <csetjmp>
#include <cstddef>
#include <cstdio>

typedef unsigned int png_uint_32;
typedef std::size_t png_size_t;
typedef unsigned char* png_bytep;
typedef const char* png_const_charp;
typedef struct png_struct_def* png_structp;
typedef struct png_info_def* png_infop;
typedef png_structp* png_structpp;
typedef png_infop* png_infopp;
typedef png_bytep* png_bytepp;
typedef void* png_voidp;
typedef void (*png_error_ptr)(png_structp, png_const_charp);

#define PNG_LIBPNG_VER_STRING "stub"
#define PNG_COLOR_TYPE_GRAY 0
#define PNG_COLOR_TYPE_RGB 2
#define PNG_COLOR_TYPE_RGB_ALPHA 6
#define PNG_COMPRESSION_TYPE_DEFAULT 0
#define PNG_FILTER_TYPE_DEFAULT 0
#define PNG_INTERLACE_NONE 0

std::jmp_buf& png_stub_jmpbuf(png_structp);
#define png_jmpbuf(p) (png_stub_jmpbuf(p))

int png_sig_cmp(const unsigned char*, png_size_t, png_size_t);
png_structp png_create_read_struct(png_const_charp, png_voidp, png_error_ptr, png_error_ptr);
png_structp png_create_write_struct(png_const_charp, png_voidp, png_error_ptr, png_error_ptr);
png_infop png_create_info_struct(png_structp);
void png_destroy_read_struct(png_structpp, png_infopp, png_infopp);
void png_destroy_write_struct(png_structpp, png_infopp);
void png_init_io(png_structp, std::FILE*);
void png_set_sig_bytes(png_structp, int);
void png_read_info(png_structp, png_infop);
png_uint_32 png_get_image_width(png_structp, png_infop);
png_uint_32 png_get_image_height(png_structp, png_infop);
int png_get_bit_depth(png_structp, png_infop);
int png_get_color_type(png_structp, png_infop);
int png_set_interlace_handling(png_structp);
void png_read_update_info(png_structp, png_infop);
png_size_t png_get_rowbytes(png_structp, png_infop);
void png_read_image(png_structp, png_bytepp);
void png_read_end(png_structp, png_infop);
void png_set_IHDR(png_structp, png_infop, png_uint_32, png_uint_32, int, int, int, int, int);
void png_write_info(png_structp, png_infop);
void png_write_row(png_structp, png_bytep);
void png_write_end(png_structp, png_infop);
#endif
